"""Launch-geometry sweep of the hop kernels on one GPU: cluster size P x hops per
block (0 = one-hop-at-a-time kernel) for each BASELINE config, device-resident
inputs, fixed filter (fresh configs) or the per-hop bank schedule (bank configs).
Prints one JSON line per point: us per hop and the §8(d) algorithmic GB/s."""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2310_00319_b200 import tvolap as T  # noqa: E402
from paper_2310_00319_b200 import workload as W  # noqa: E402
from paper_2310_00319_b200.tvolap import TvolapBankEngine, TvolapEngine, partition  # noqa: E402

HOPS = {"C1": 3750, "C2": 1024, "C3": 512, "C4": 128, "C5": 1024}


def run(name, Ps, JHs, reps=3, period=0, exchange=False, switching=False):
    cfg = W.CONFIGS[name]
    H, L, S = HOPS[name], cfg.hop, cfg.sources
    lib = T.lib()
    x = torch.empty((S, H * L), device="cuda")
    T._check(lib.tvolap_gen_white_device(0, cfg.seed, 0, S, 0, H * L, ctypes.c_void_p(x.data_ptr()), H * L))
    out = torch.empty((cfg.lanes, H * L), device="cuda")
    sched = None
    if cfg.mode == "bank":
        bank = torch.from_numpy(W.bank_irs(cfg)).cuda()
        sched_h = W.schedule(cfg, 0, H)
        sched = torch.from_numpy(sched_h).cuda()
        distinct = float(np.mean([np.unique(r).size for r in sched_h[:256]]))
        eng = TvolapBankEngine(bank, L, S, min_partitions=cfg.partitions)
    else:
        eng = TvolapEngine(partition(W.fresh_irs(cfg, 0)[:, 0, :].T, L, cfg.partitions))
        distinct = S
        irs = torch.from_numpy(np.stack([W.fresh_irs(cfg, k)[:, 0, :] for k in range(2)])).cuda() if exchange else None

    def step():
        if switching:  # one tvolap_process_switching call (in-kernel K4)
            eng.process_switching(x, [irs[k & 1] for k in range(-(-H // period))], period, out=out)
            return
        if not period:
            eng.process_hops(x, out=out, schedule=sched)
            return
        for h0 in range(0, H, period):
            if exchange:
                eng.exchange_ir(irs[(h0 // period) & 1])
            sl = slice(h0 * L, min(H, h0 + period) * L)
            eng.process_hops(x[:, sl], out=out[:, sl], schedule=None if sched is None else sched[h0:h0 + period])
    st = torch.cuda.Stream()
    eng.set_stream(st.cuda_stream)
    bph = W.bytes_per_hop(cfg, distinct_filters=distinct)
    for P in Ps:
        if P > L:
            continue
        for jh in JHs:
            try:
                eng.set_launch_config(P, 0)
                if jh == 0:
                    eng.set_block_config(0, 1 << 30)
                else:
                    eng.set_block_config(2 * jh, 2)
            except (T.InvalidConfigurationError, T.CudaError) as e:
                print(json.dumps({"cfg": name, "P": P, "J": 2 * jh, "skip": str(e)}), flush=True)
                continue
            try:
                step()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                for _ in range(reps):
                    step()
                b.record(st)
                b.synchronize()
                ms = a.elapsed_time(b) / reps
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"cfg": name, "P": P, "J": 2 * jh, "error": str(e)}), flush=True)
                continue
            j, bm, q = eng.block_config()
            print(json.dumps({"cfg": name, "P": P, "J": 2 * jh, "Q": q, "period": period, "exchange": exchange,
                              "switching": switching,
                              "us_per_hop": 1e3 * ms / H,
                              "GBps_alg": bph * H / (ms / 1e3) / 1e9, "frac": bph * H / (ms / 1e3) / 1e9 / 6542.1}),
                  flush=True)


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--P", type=int, nargs="*", default=[1, 2, 4, 8])
    ap.add_argument("--J", type=int, nargs="*", default=[0, 2, 4, 8, 16], help="hops per block (0 = streaming)")
    ap.add_argument("--hops", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--period", type=int, default=0, help="hops per process_hops call (0 = one call)")
    ap.add_argument("--exchange", action="store_true", help="exchange_filter before every call (fresh configs)")
    ap.add_argument("--switching", action="store_true", help="one process_switching call per pass (fresh configs)")
    a = ap.parse_args()
    for n in a.configs:
        if a.hops:
            HOPS[n] = a.hops
        run(n, a.P, [j // 2 for j in a.J], reps=a.reps, period=a.period, exchange=a.exchange or a.switching,
            switching=a.switching)
