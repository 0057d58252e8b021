"""Period tiles (csrc/tvolap_wide.cu wide_period_kernel): a device-resident process_switching call
whose filter periods are <= 8 hops (C4: L=512, M=256, a fresh IR every 8 hops) runs as K1 for all
hops + one CTA per (lane, period) that transforms the period's set in shared-memory partition
groups (IR slices by cp.async.bulk + mbarrier), MACs against the delay line and runs K5 + the
overlap-add. It must match the exchange_filter + process_hops loop of the hop-blocked kernel to
fp32 rounding, the reference engine (oracle/_ref) within the north-star bound, and hand the same
state to later calls."""
import numpy as np
import pytest
import torch

from paper_2310_00319_b200 import tvolap as T
from paper_2310_00319_b200 import workload as W
from parity import TOL, oracle_config, rel_err

pytestmark = pytest.mark.gpu


def _loop(eng, x, dirs, period, hop):
    n = x.shape[1] // hop
    out = torch.empty_like(x)
    for k in range(-(-n // period)):
        if dirs[k] is not None:
            eng.exchange_ir(dirs[k])
        sl = slice(k * period * hop, min(n, (k + 1) * period) * hop)
        eng.process_hops(x[:, sl], out=out[:, sl])
    return out


def _rel(a, b):
    a, b = a.cpu().numpy().astype(np.float64), b.cpu().numpy().astype(np.float64)
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("hop,S,taps,n_hops,period,none_at,pre", [
    (512, 3, 256 * 1024, 8 * 6 + 5, 8, (), 0),          # C4 geometry, ragged 5-hop final period
    (512, 2, 256 * 1024, 8 * 5, 8, (0, 2), 3),          # first tile and a middle one on the active set
    (512, 2, 64 * 1024 - 512, 8 * 4 + 3, 8, (), 1),     # M = 64, last group's taps partly past the IR
    (512, 3, 128 * 1024, 6 * 7, 6, (3,), 2),            # 6-hop periods
    (256, 3, 64 * 512, 8 * 6, 8, (), 1),                # 512-point transforms (G = 8)
    (512, 2, 32 * 1024, 3 * 12, 3, (), 0),              # shortest tile (3 hops)
    (256, 3, 64 * 512, 16 * 5 + 7, 16, (2,), 1),        # C2 geometry (16-hop periods: wide_mac_kernel's L2 slots)
    (256, 2, 32 * 512 - 256, 12 * 4, 12, (0,), 2),      # 12-hop periods (wide_mac_kernel)
])
def test_period_tiles_equal_exchange_loop(hop, S, taps, n_hops, period, none_at, pre):
    g = np.random.default_rng(hop + S + taps + period)
    nsw = -(-n_hops // period)
    irs = [None if k in none_at else torch.from_numpy(g.standard_normal((S, taps)).astype(np.float32) * 0.02).cuda()
           for k in range(nsw)]
    ir0 = g.standard_normal((taps, S)) * 0.02
    x = torch.from_numpy(g.uniform(-1, 1, (S, (pre + n_hops) * hop)).astype(np.float32)).cuda()
    a = T.TvolapEngine(T.partition(ir0, hop))
    b = T.TvolapEngine(T.partition(ir0, hop))
    b.set_tuning("wide", 0)
    if pre:
        a.process_hops(x[:, : pre * hop])
        b.process_hops(x[:, : pre * hop])
    xs = x[:, pre * hop:]
    ya = a.process_switching(xs, irs, period)
    yb = _loop(b, xs, irs, period, hop)
    a.synchronize()
    b.synchronize()
    assert a.wide_passes() >= 1 and b.wide_passes() == 0
    assert _rel(ya, yb) <= 1e-5
    # the state handed on: delay line, carry, history and the active set (the last IR)
    za, zb = a.process_hops(x[:, : 24 * hop]), b.process_hops(x[:, : 24 * hop])
    a.synchronize()
    b.synchronize()
    assert _rel(za, zb) <= 1e-5
    assert a.op_counts() == b.op_counts()


def test_period_tiles_off_is_the_slot_path():
    """wide_period=0 keeps the global-scratch fused K4 (wide_mac_kernel): same results to rounding."""
    hop, S, taps, n = 512, 2, 64 * 1024, 40
    g = np.random.default_rng(7)
    irs = [torch.from_numpy(g.standard_normal((S, taps)).astype(np.float32) * 0.02).cuda() for _ in range(5)]
    ir0 = g.standard_normal((taps, S)) * 0.02
    x = torch.from_numpy(g.uniform(-1, 1, (S, n * hop)).astype(np.float32)).cuda()
    a = T.TvolapEngine(T.partition(ir0, hop))
    b = T.TvolapEngine(T.partition(ir0, hop))
    b.set_tuning("wide", 2)
    b.set_tuning("wide_period", 0)
    ya, yb = a.process_switching(x, irs, 8), b.process_switching(x, irs, 8)
    a.synchronize()
    b.synchronize()
    assert a.wide_passes() == 1 and b.wide_passes() == 1
    assert _rel(ya, yb) <= 1e-5


def test_c4_device_path_vs_reference():
    """C4 as the bench runs it (process_switching on device buffers: the period tiles), 8 lanes over
    1100 hops (ring of 264 slots wrapped, 138 switches) against the reference engine."""
    cfg = W.CONFIGS["C4"]
    S, n, L = 8, 1100, cfg.hop
    x = torch.from_numpy(W.white(cfg, 0, S, 0, n * L)).cuda()
    nsw = -(-n // cfg.period)
    irs = [None] + [torch.from_numpy(np.ascontiguousarray(W.fresh_irs(cfg, k, 0, S)[:, 0, :])).cuda()
                    for k in range(1, nsw)]
    eng = T.TvolapEngine(T.partition(W.fresh_irs(cfg, 0, 0, S)[:, 0, :].T, L, cfg.partitions))
    y = eng.process_switching(x, irs, cfg.period)
    eng.synchronize()
    assert eng.wide_passes() >= 1
    ref = oracle_config(cfg, n, sources=S)
    err = rel_err(y.cpu().numpy(), ref)
    assert err <= TOL, err


def test_c2_device_path_vs_reference():
    """C2 as the bench runs it (process_switching on device buffers: the time-parallel pass with K4
    fused into L2 scratch slots), 6 lanes
    over 400 hops (25 switches, ring wrapped) against the reference engine."""
    cfg = W.CONFIGS["C2"]
    S, n, L = 6, 400, cfg.hop
    x = torch.from_numpy(W.white(cfg, 0, S, 0, n * L)).cuda()
    nsw = -(-n // cfg.period)
    irs = [None] + [torch.from_numpy(np.ascontiguousarray(W.fresh_irs(cfg, k, 0, S)[:, 0, :])).cuda()
                    for k in range(1, nsw)]
    eng = T.TvolapEngine(T.partition(W.fresh_irs(cfg, 0, 0, S)[:, 0, :].T, L, cfg.partitions))
    y = eng.process_switching(x, irs, cfg.period)
    eng.synchronize()
    assert eng.wide_passes() >= 1
    ref = oracle_config(cfg, n, sources=S)
    err = rel_err(y.cpu().numpy(), ref)
    assert err <= TOL, err


@pytest.mark.parametrize("case", ["taps_not_multiple_of_4", "ir_not_16B_aligned", "bit_identical_mode"])
def test_period_tiles_fall_back(case):
    """Where the bulk copies cannot take the IR slices (tap count not a multiple of 4, a set not
    16-byte aligned) or the caller asked for the hop kernels' transforms (wide_warp_fft = 0), C4
    geometry runs on wide_mac_kernel instead — same results to fp32 rounding."""
    hop, S, n, period = 512, 2, 40, 8
    taps = 64 * 1024 - (2 if case == "taps_not_multiple_of_4" else 0)
    g = np.random.default_rng(3)
    irs = []
    for _ in range(n // period):
        h = torch.from_numpy(g.standard_normal((S, taps + 1)).astype(np.float32) * 0.02).cuda()
        irs.append(h[:, 1:] if case == "ir_not_16B_aligned" else h[:, :taps].contiguous())
    if case == "ir_not_16B_aligned":  # a dense (lanes, taps) view starting one float in
        flat = torch.from_numpy(g.standard_normal(S * taps + 1).astype(np.float32) * 0.02).cuda()
        irs = [flat[1:].view(S, taps) for _ in irs]
    ir0 = g.standard_normal((taps, S)) * 0.02
    x = torch.from_numpy(g.uniform(-1, 1, (S, n * hop)).astype(np.float32)).cuda()
    a = T.TvolapEngine(T.partition(ir0, hop))
    b = T.TvolapEngine(T.partition(ir0, hop))
    b.set_tuning("wide", 0)
    if case == "bit_identical_mode":
        a.set_tuning("wide_warp_fft", 0)
    ya = a.process_switching(x, irs, period)
    yb = _loop(b, x, irs, period, hop)
    a.synchronize()
    b.synchronize()
    assert a.wide_passes() >= 1
    assert _rel(ya, yb) <= 1e-5
