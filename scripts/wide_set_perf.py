import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2310_00319_b200 import tvolap as T
for mode in ["0", "1"]:
    g = np.random.default_rng(0)
    S, hop, taps, n = 2, 256, 32768, 5625
    eng = T.TvolapEngine(T.partition(g.standard_normal((taps, S)) * 0.01, hop))
    eng.set_tuning("wide", int(mode))
    x = torch.from_numpy(g.uniform(-1, 1, (S, n * hop)).astype(np.float32)).cuda()
    out = torch.empty_like(x)
    torch.cuda.synchronize()
    for _ in range(2): eng.reset(); eng.process_hops(x, out=out)
    eng.synchronize()
    t = time.time()
    for _ in range(5): eng.reset(); eng.process_hops(x, out=out)
    eng.synchronize()
    dt = (time.time() - t) / 5
    print("WIDE", mode, "2ch x 30 s (L=256, M=64):", round(dt * 1e3, 2), "ms per pass", "%.3g ch-samples/s" % (S * n * hop / dt), "passes", eng.wide_passes())
