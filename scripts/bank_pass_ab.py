"""A/B of the bank pass's partition-group count Q (tuning "bank_pass_q") on C3 / C5: one full pass
per step on device buffers, CUDA events, same box; prints one JSON line per (config, Q)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2310_00319_b200 import drive  # noqa: E402
from paper_2310_00319_b200 import workload as W  # noqa: E402

for name, qs in (("C5", [4, 8, 16]), ("C3", [2, 4, 8])):
    cfg = W.CONFIGS[name]
    H, L, S = cfg.hops, cfg.hop, cfg.sources
    x = torch.from_numpy(W.white(cfg, 0, S, 0, H * L)).cuda()
    sched = torch.from_numpy(W.schedule(cfg, 0, H)).cuda()
    out = torch.empty((S * cfg.ears, H * L), device="cuda")
    for q in qs:
        eng = drive.make_engine(cfg)
        eng.set_tuning("bank_pass_q", q)
        for _ in range(2):
            eng.reset()
            eng.process_hops(x, out=out, schedule=sched)
        eng.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = torch.cuda.current_stream()
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(3):
            eng.reset()
            eng.process_hops(x, out=out, schedule=sched)
        eng.synchronize()
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        print(json.dumps({"config": name, "Q": q, "ms_per_pass": ms, "us_per_hop": 1e3 * ms / H,
                          "value": S * cfg.ears * H * L / (ms / 1e3)}), flush=True)
        del eng
