"""Multi-rank run of the CUDA engine: 2 ranks (gloo rendezvous on 127.0.0.1),
each driving the engine on its own contiguous channel range — the strong-scaling split bench.py
uses — on the one GPU of this box (the ranks share no kernels and never wait on each other's
device work). Rank outputs are gathered and checked against the reference; C3's stereo mix is
each rank's partial mix (tvolap_mix_allreduce) summed across ranks, against the reference mix."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_HOPS = 80


def _worker(rank, world, port, out_dir):
    import ctypes
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    import torch
    import torch.distributed as dist

    from paper_2310_00319_b200 import drive, shard
    from paper_2310_00319_b200 import tvolap as T
    from paper_2310_00319_b200 import workload as W

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    for name, total in (("C5", 128), ("C3", 64)):
        cfg = W.CONFIGS[name].scaled(sources=total)
        lane0, S = shard.strong_lanes(total, rank, world)
        eng = drive.make_engine(cfg, lane0, S)
        L = cfg.hop
        x = torch.from_numpy(W.white(cfg, lane0, S, 0, N_HOPS * L)).cuda()
        sched = torch.from_numpy(W.schedule(cfg, 0, N_HOPS, lane0, S)).cuda()
        y = eng.process_hops(x, schedule=sched)
        eng.synchronize()
        assert eng.wide_passes() >= 1  # the bank pass on each rank's shard
        np.save(os.path.join(out_dir, f"{name}_{rank}.npy"), y.cpu().numpy())
        if cfg.mix:
            mix = torch.empty((cfg.ears, N_HOPS * L), device="cuda")
            T._check(T.lib().tvolap_mix_allreduce(0, S, cfg.ears, N_HOPS * L, ctypes.c_void_p(y.data_ptr()), N_HOPS * L,
                                                  ctypes.c_void_p(mix.data_ptr()), N_HOPS * L, None, None))
            torch.cuda.synchronize()
            m = mix.cpu()
            shard.mix_allreduce(m)  # gloo here; NCCL (tvolap_mix_allreduce's comm) across GPUs
            if rank == 0:
                np.save(os.path.join(out_dir, f"{name}_mix.npy"), m.numpy())
            # the fused peer-memory mix: each rank's kernel stores its partial into both ranks'
            # gather buffers (cudaIpc-mapped; P2P over NVLink across GPUs), rank-ordered sums
            grp = shard.MixGroup(0, cfg.ears, N_HOPS * L)
            pm = torch.empty((cfg.ears, N_HOPS * L), device="cuda")
            grp.allreduce(y, S, N_HOPS * L, pm)
            np.save(os.path.join(out_dir, f"{name}_pmix_{rank}.npy"), pm.cpu().numpy())
            grp.close()
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_strong_split_matches_reference(tmp_path):
    import socket

    import torch.multiprocessing as mp

    from paper_2310_00319_b200 import workload as W
    from parity import TOL, oracle_config, rel_err

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    for name, total in (("C5", 128), ("C3", 64)):
        cfg = W.CONFIGS[name].scaled(sources=total)
        y = np.concatenate([np.load(tmp_path / f"{name}_{r}.npy") for r in range(2)])
        assert y.shape[0] == total * cfg.ears
        ref = oracle_config(cfg, N_HOPS)
        assert rel_err(y, ref) <= TOL, name
        if cfg.mix:
            mref = ref.reshape(total, cfg.ears, -1).sum(0)
            assert rel_err(np.load(tmp_path / f"{name}_mix.npy"), mref) <= TOL
            # peer-memory mix: the same bits on both ranks, = the rank-ordered fp32 sum of the
            # per-rank source-ordered partials, and within the north-star bound of the reference mix
            pm = [np.load(tmp_path / f"{name}_pmix_{r}.npy") for r in range(2)]
            assert np.array_equal(pm[0], pm[1])
            want = None
            for r in range(2):
                lane0, S = (0, total // 2) if r == 0 else (total // 2, total - total // 2)
                part = np.zeros((cfg.ears, y.shape[1]), np.float32)
                for s_ in range(lane0, lane0 + S):
                    part += y[s_ * cfg.ears: (s_ + 1) * cfg.ears]
                want = part if want is None else want + part
            assert np.array_equal(pm[0], want)
            assert rel_err(pm[0], mref) <= TOL
