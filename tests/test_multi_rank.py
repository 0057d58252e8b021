"""World-size-2 gloo tests of the multi-GPU host logic (run on CPU): lane sharding and the C3
stereo-mix all-reduce. Each rank convolves its shard with the CPU oracle (the GPU kernel's
per-lane results are independent of the shard, which the GPU tests check against the same
oracle), then the partial mixes are all-reduced and compared with a single-process mix."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2310_00319_b200 import shard
from paper_2310_00319_b200 import workload as W

CFG = W.CONFIGS["C3"].scaled(hop=16, partitions=4, sources=6, n_bank=5, seconds=0.02)
N_HOPS = 24


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mix_of(lane0, n):
    cfg = CFG
    x = np.stack([W.white(cfg, lane0 + s, 1, 0, N_HOPS * cfg.hop, dtype=np.float64)[0] for s in range(n)])
    bank = W.bank_irs(cfg, dtype=np.float64)
    sched = W.schedule(cfg, 0, N_HOPS, lane0, n)
    _, y = O.run_workload(cfg.hop, cfg.partitions, n, cfg.ears, N_HOPS, x, 1, bank_ir=bank, schedule=sched,
                          threads=2)
    return y.reshape(n, cfg.ears, -1).sum(0)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lane0, n = shard.strong_lanes(CFG.sources, rank, world)
    mix = torch.from_numpy(_mix_of(lane0, n))
    shard.mix_allreduce(mix)
    t = shard.max_over_ranks(float(rank + 1))
    if rank == 0:
        np.save(out, mix.numpy())
        np.save(out + ".t.npy", np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


def test_lane_ranges_cover_exactly():
    for total in (1, 5, 64, 1024):
        for world in (1, 2, 3, 8):
            ranges = [shard.strong_lanes(total, r, world) for r in range(world)]
            assert sum(n for _, n in ranges) == total
            assert all(ranges[i][0] + ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    assert shard.weak_lanes(64, 3) == (192, 64)


@pytest.mark.timeout(300)
def test_two_rank_mix_allreduce_matches_single_process(tmp_path):
    out = str(tmp_path / "mix.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    ref = _mix_of(0, CFG.sources)
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.load(out + ".t.npy")[0] == 2.0  # max over ranks
