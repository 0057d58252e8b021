"""Per-hop copy latencies of the one-hop process() path (C5 sizes): pinned 512 KB H2D / D2H and a
32 KB pageable H2D, each timed alone with CUDA events on one stream (median of 200)."""
import numpy as np
import torch

s = torch.cuda.Stream()
def timed(fn, n=200):
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s); fn(); b.record(s)
        b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))
for nb in (32 << 10, 512 << 10, 2 << 20):
    hp = torch.empty(nb // 4, dtype=torch.float32, pin_memory=True)
    hq = torch.empty(nb // 4, dtype=torch.float32)
    d = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
    print(f"{nb >> 10:5d} KB  pinned H2D {timed(lambda: d.copy_(hp, non_blocking=True)):7.1f} us  "
          f"pinned D2H {timed(lambda: hp.copy_(d, non_blocking=True)):7.1f} us  "
          f"pageable H2D {timed(lambda: d.copy_(hq, non_blocking=True)):7.1f} us  empty {timed(lambda: None):5.1f} us")
