"""Per-phase SM-cycle breakdown of the hop-blocked kernel (diagnostic build with
TVOLAP_PHASE_PROF; build it here with `python scripts/phase_prof.py --build`).

Runs one config's throughput path (device-resident inputs, optional exchange every
`--period` hops) and prints average cycles per CTA per block for each phase."""
import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2310_00319_b200 import _build  # noqa: E402

NAMES = ["input_wait", "fwd_fft+ring", "sync_ring", "mac", "reduce", "sync_y", "gather+ifft", "sync_td", "ola",
         "hist", "sync_end", "prologue"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--hops", type=int, default=512)
    ap.add_argument("--period", type=int, default=0)
    ap.add_argument("--exchange", action="store_true")
    ap.add_argument("--switching", action="store_true", help="one process_switching call (in-kernel K4)")
    a = ap.parse_args()
    path = _build.build_variant("prof", ["TVOLAP_PHASE_PROF"])
    if a.build:
        return
    import numpy as np
    import torch

    from paper_2310_00319_b200 import tvolap as T
    from paper_2310_00319_b200 import workload as W
    T._LIB_PATH = path
    lib = T.lib()
    lib.tvolap_phase_counters.restype = ctypes.c_int
    lib.tvolap_phase_counters.argtypes = [ctypes.c_void_p, ctypes.c_int]
    cfg = W.CONFIGS[a.config]
    H, L, S = a.hops, cfg.hop, cfg.sources
    x = torch.empty((S, H * L), device="cuda")
    T._check(lib.tvolap_gen_white_device(0, cfg.seed, 0, S, 0, H * L, ctypes.c_void_p(x.data_ptr()), H * L))
    out = torch.empty((cfg.lanes, H * L), device="cuda")
    sched = None
    if cfg.mode == "bank":
        bank = torch.from_numpy(W.bank_irs(cfg)).cuda()
        sched = torch.from_numpy(W.schedule(cfg, 0, H)).cuda()
        eng = T.TvolapBankEngine(bank, L, S, min_partitions=cfg.partitions)
    else:
        eng = T.TvolapEngine(T.partition(W.fresh_irs(cfg, 0)[:, 0, :].T, L, cfg.partitions))
        irs = torch.from_numpy(np.stack([W.fresh_irs(cfg, k)[:, 0, :] for k in range(2)])).cuda()
    period = a.period or H

    def step():
        if a.switching:
            eng.process_switching(x, [irs[k & 1] for k in range(-(-H // period))], period, out=out)
            return
        for h0 in range(0, H, period):
            if a.exchange:
                eng.exchange_ir(irs[(h0 // period) & 1])
            sl = slice(h0 * L, min(H, h0 + period) * L)
            eng.process_hops(x[:, sl], out=out[:, sl], schedule=None if sched is None else sched[h0:h0 + period])

    buf = (ctypes.c_ulonglong * 16)()
    step()
    lib.tvolap_phase_counters(buf, 16)
    step()
    assert lib.tvolap_phase_counters(buf, 16) == 0
    blocks = max(1, buf[12])
    row = {n: round(buf[i] / blocks, 1) for i, n in enumerate(NAMES)}
    row["total"] = round(sum(buf[i] for i in range(11)) / blocks, 1)
    print(json.dumps({"cfg": a.config, "period": a.period, "exchange": a.exchange,
                      "block_config": list(eng.block_config()), "cta_blocks": blocks,
                      "cycles_per_cta_block": row}))


if __name__ == "__main__":
    main()
