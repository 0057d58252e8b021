"""GPU-side launch timeline of the hop-blocked kernel and the side-stream K4 (diagnostic build
with TVOLAP_PHASE_PROF): globaltimer at the first CTA's start and the last CTA's end of every
launch, for a fresh-IR config driven as bench.py does (exchange_ir + process_hops per period)."""
import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2310_00319_b200 import _build  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--switches", type=int, default=64)
    ap.add_argument("--no-exchange", action="store_true")
    a = ap.parse_args()
    path = _build.build_variant("prof", ["TVOLAP_PHASE_PROF"])
    import numpy as np
    import torch

    from paper_2310_00319_b200 import tvolap as T
    from paper_2310_00319_b200 import workload as W
    T._LIB_PATH = path
    lib = T.lib()
    cfg = W.CONFIGS[a.config]
    L, S, per = cfg.hop, cfg.sources, cfg.period
    H = per * a.switches
    x = torch.empty((S, H * L), device="cuda")
    T._check(lib.tvolap_gen_white_device(0, cfg.seed, 0, S, 0, H * L, ctypes.c_void_p(x.data_ptr()), H * L))
    out = torch.empty((S, H * L), device="cuda")
    eng = T.TvolapEngine(T.partition(W.fresh_irs(cfg, 0)[:, 0, :].T, L, cfg.partitions))
    irs = torch.from_numpy(np.stack([W.fresh_irs(cfg, k)[:, 0, :] for k in range(2)])).cuda()
    st = torch.cuda.Stream()
    eng.set_stream(st.cuda_stream)

    def run():
        for k in range(a.switches):
            if not a.no_exchange:
                eng.exchange_ir(irs[k & 1])
            eng.process_hops(x[:, k * per * L:(k + 1) * per * L], out=out[:, k * per * L:(k + 1) * per * L])

    n = 4096
    buf = (ctypes.c_ulonglong * (2 * n * 2))()
    cnt = (ctypes.c_uint * 2)()
    import time
    run()
    lib.tvolap_timeline(buf, n, cnt)
    torch.cuda.synchronize()
    t_host = time.perf_counter()
    run()
    t_host = time.perf_counter() - t_host
    assert lib.tvolap_timeline(buf, n, cnt) == 0
    tl = np.frombuffer(buf, dtype=np.uint64).reshape(2, n, 2).astype(np.float64)
    nh, nk = cnt[0], cnt[1]
    hop, k4 = tl[0, :nh], tl[1, :nk]
    t0 = hop[0, 0]
    rows = []
    for i in range(min(nh, 12)):
        r = {"hop_begin": (hop[i, 0] - t0) / 1e3, "hop_end": (hop[i, 1] - t0) / 1e3}
        if i < nk:
            r.update(k4_begin=(k4[i, 0] - t0) / 1e3, k4_end=(k4[i, 1] - t0) / 1e3)
        rows.append({k: round(v, 2) for k, v in r.items()})
    dur = (hop[:, 1] - hop[:, 0]) / 1e3
    gaps = (hop[1:, 0] - hop[:-1, 1]) / 1e3
    summ = {"cfg": a.config, "exchange": not a.no_exchange, "hop_launches": int(nh), "k4_launches": int(nk),
            "hop_us_mean": float(dur.mean()), "gap_us_mean": float(gaps.mean()),
            "period_us_mean": float((hop[-1, 1] - hop[0, 0]) / 1e3 / nh),
            "host_enqueue_us_per_period": 1e6 * t_host / a.switches}
    if nk:
        kd = (k4[:, 1] - k4[:, 0]) / 1e3
        summ["k4_us_mean"] = float(kd.mean())
    print(json.dumps(summ))
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
