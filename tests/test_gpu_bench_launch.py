"""bench.py's multi-GPU launcher end to end on the one GPU of this box: `--gpus 2` re-launches the
script under torch.distributed.run (one process per rank), `--one-gpu` puts both ranks on cuda:0
over gloo (NCCL needs a GPU per rank), the strong split gives each rank half of the channels, the
timing is the max over ranks, and C3's stereo mix runs through the fused peer-memory path
(cudaIpc-mapped gather buffers between the two processes). Each rank's dumped outputs are checked
against the reference engine; the mix must be bit-identical on both ranks."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2310_00319_b200 import workload as W
from parity import TOL, oracle_config, rel_err

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _launch(cfg_name, hops, dump):
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--one-gpu", "--config", cfg_name, "--hops",
           str(hops), "--steps", "1", "--warmup", "3", "--no-cpu", "--no-e2e", "--latency-hops", "0", "--dump",
           str(dump)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


def _gather(dump):
    parts, shards = [], []
    for rk in range(2):
        parts.append(np.load(dump / f"out_{rk}.npy"))
        shards.append(json.loads((dump / f"shard_{rk}.json").read_text()))
    return parts, shards


def test_bench_two_ranks_c5(tmp_path):
    line = _launch("C5", 48, tmp_path)
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["sources_per_gpu"] == 2048
    parts, shards = _gather(tmp_path)
    assert [s["lane0"] for s in shards] == [0, 2048] and [s["sources"] for s in shards] == [2048, 2048]
    y = np.concatenate(parts)
    cfg = W.CONFIGS["C5"]
    subset = list(range(0, 4096, 64)) + [2047, 2048]
    ref = oracle_config(cfg, 48, subset=subset)
    assert rel_err(y[subset], ref) <= TOL


def test_bench_two_ranks_c3_peer_mix(tmp_path):
    line = _launch("C3", 24, tmp_path)
    assert line["n_gpus"] == 2 and line["mix_path"].startswith("peer memory")
    parts, shards = _gather(tmp_path)
    m0, m1 = np.load(tmp_path / "mix_0.npy"), np.load(tmp_path / "mix_1.npy")
    assert np.array_equal(m0, m1)
    cfg = W.CONFIGS["C3"]
    y = np.concatenate(parts)
    ref = oracle_config(cfg, 24)  # all 1024 sources x 2 ears
    assert rel_err(y, ref) <= TOL
    assert rel_err(m0, ref.reshape(1024, 2, -1).sum(0)) <= TOL
