import os, sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
from test_gpu_wide import _case, _loop
from paper_2310_00319_b200 import tvolap as T

def run(hop, S, taps, n, period, pre):
    ir0, x, dirs = _case(hop, S, taps, n, period)
    os.environ["TVOLAP_WIDE"] = "2"; a = T.TvolapEngine(T.partition(ir0, hop))
    os.environ["TVOLAP_WIDE"] = "0"; b = T.TvolapEngine(T.partition(ir0, hop))
    if pre:
        a.process_hops(x[:, :pre*hop]); b.process_hops(x[:, :pre*hop])
    ya = a.process_switching(x, dirs, period).cpu().numpy(); yb = _loop(b, x, dirs, period, hop).cpu().numpy()
    d = np.abs(ya - yb).reshape(S, n, hop).max(axis=(0, 2))
    bad = np.nonzero(d)[0]
    print(hop, S, taps, n, period, pre, "bad hops:", bad[:20], len(bad), flush=True)

for args in [(32, 6, 1024, 90, 17, 2), (32, 6, 1024, 90, 16, 2), (32, 6, 1024, 90, 17, 0), (32, 1, 1024, 90, 17, 0),
             (64, 6, 2048, 90, 17, 2), (32, 6, 2048, 90, 17, 2), (32, 6, 512, 90, 17, 2)]:
    run(*args)
