"""One-hop kernel time against the number of sources (C3 geometry: L = 128, M = 128, 2 ears, bank of 256):
does the launch time follow the waves of resident CTAs (4 per SM x 148 = 592) or the bytes?
python scripts/hop_waves.py  ->  one line per S: kernel us, DRAM-compulsory GB/s."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2310_00319_b200 import tvolap as T  # noqa: E402

hop, M, ears, n_bank = 128, 128, 2, 256
g = np.random.default_rng(1)
taps = 2 * hop * M  # partitions are 2L taps long (hop-2 overlap-add, 4L transforms)
bank = (g.standard_normal((n_bank, ears, taps)) * np.exp(-np.arange(taps) / (taps / 6))).astype(np.float32)
for S in (148, 296, 444, 592, 740, 888, 1024, 1184, 1776):
    e = T.TvolapBankEngine(bank, hop, S)
    x = g.uniform(-1, 1, (hop, S)).astype(np.float32)
    sels = g.integers(0, n_bank, (120, S)).astype(np.int32)  # a fresh selection every hop, as in the bench
    sel = sels[-1]
    for h in range(20):
        e.select_bank(sels[h])
        e.process(x)
    e.set_profiling(True)
    for h in range(20, 120):
        e.select_bank(sels[h])
        e.process(x)
    ms, n = e.kernel_time()
    e.set_profiling(False)
    us = ms / n * 1e3
    distinct = len(np.unique(sel))
    byts = S * M * hop * 2 * 8 + distinct * ears * M * hop * 2 * 8  # delay-line rows + distinct filter rows (2L packed bins x 8 B)
    print(f"S {S:5d}  kernel {us:7.1f} us  waves {S / 592:.2f}  {byts / us / 1e3:7.1f} GB/s  us per 592-wave {us / max(1, -(-S // 592)):.1f}", flush=True)
    del e

# the bench's latency-leg call on the same geometry: pinned host tensors through tvolap_process (in place / with copies)
import ctypes  # noqa: E402

import torch  # noqa: E402

S = 1024
lib = T.lib()
for zc, own_stream in ((1, False), (0, False), (1, True), (0, True)):
    e = T.TvolapBankEngine(bank, hop, S)
    e.set_tuning("zero_copy", zc)
    st = torch.cuda.Stream()
    if own_stream:
        e.set_stream(st.cuda_stream)
    xin = torch.empty((S, hop), dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
    yout = torch.empty((S * ears, hop), dtype=torch.float32, pin_memory=True)
    sels = g.integers(0, n_bank, (120, S)).astype(np.int32)
    for h in range(120):
        if h == 20:
            e.set_profiling(True)
        e.select_bank(sels[h])
        T._check(lib.tvolap_process(e._h, ctypes.c_void_p(xin.data_ptr()), hop, hop, S, ctypes.c_void_p(yout.data_ptr()), hop))
        e.synchronize()
    ms, n = e.kernel_time()
    print(f"S {S} pinned tensors zero_copy={zc} torch stream={own_stream}: kernel {ms / n * 1e3:.1f} us over {n} launches", flush=True)
    del e
