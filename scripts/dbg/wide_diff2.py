import os, sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
from test_gpu_wide import _case, _loop
from paper_2310_00319_b200 import tvolap as T
import oracle as O

def oracle_run(ir0, x, dirs, hop, period, n):
    xs = x.cpu().numpy().astype(np.float64)
    eng = O.Engine(O.partition(ir0.astype(np.float32).astype(np.float64), hop))
    ref = []
    for h in range(n):
        if h % period == 0 and dirs[h // period] is not None:
            eng.exchange_filter(O.partition(dirs[h // period].cpu().numpy().T.astype(np.float64), hop, eng.partition_count()))
        ref.append(eng.process(xs[:, h * hop:(h + 1) * hop].T))
    return np.concatenate(ref).T

def run(hop, S, taps, n, period, env=None):
    ir0, x, dirs = _case(hop, S, taps, n, period)
    for k, v in (env or {}).items(): os.environ[k] = v
    os.environ["TVOLAP_WIDE"] = "2"; a = T.TvolapEngine(T.partition(ir0, hop))
    os.environ["TVOLAP_WIDE"] = "0"; b = T.TvolapEngine(T.partition(ir0, hop))
    for k in (env or {}): del os.environ[k]
    ya = a.process_switching(x, dirs, period).cpu().numpy(); yb = _loop(b, x, dirs, period, hop).cpu().numpy()
    ref = oracle_run(ir0, x, dirs, hop, period, n)
    sc = np.abs(ref).max()
    ea = np.abs(ya - ref).reshape(S, n, hop).max(axis=(0, 2)) / sc
    eb = np.abs(yb - ref).reshape(S, n, hop).max(axis=(0, 2)) / sc
    print(hop, S, taps, n, period, env, "wide err", ea.max(), np.nonzero(ea > 1e-4)[0][:8], "blocked err", eb.max(),
          "bitexact", np.array_equal(ya, yb), "geom", b.block_config() if hasattr(b, "block_config") else None, flush=True)

if __name__ == "__main__": run(32, 6, 1024, 90, 17)
#run(32, 6, 1024, 90, 17, {"TVOLAP_PB": "1"})
#run(64, 6, 2048, 90, 17)
#run(128, 6, 2048, 90, 17)
#run(32, 1, 1024, 40, 16)
