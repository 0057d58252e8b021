"""Time-parallel pass (csrc/tvolap_wide.cu): a device-resident tvolap_process_switching call run
as K4-for-all-sets + K1-for-all-hops + (lane, tile) MAC/inverse CTAs + OLA fix-up must equal the
exchange_filter + process_hops loop it stands for (hop-blocked kernel) and leave the engine in the
same state (delay line, carry, history, active set): bit for bit with the hop kernels' Stockham
transforms (TVOLAP_WIDE_WARPFFT=0), to fp32 rounding with the default warp-per-frame transforms."""
import numpy as np
import pytest

import oracle as O
from paper_2310_00319_b200 import tvolap as T

pytestmark = pytest.mark.gpu


def _case(hop, S, taps, n_hops, period, none_at=(), seed=0):
    import torch

    g = np.random.default_rng(seed)
    nsw = -(-n_hops // period)
    irs = [None if k in none_at else g.standard_normal((S, taps)).astype(np.float32) * 0.05 for k in range(nsw)]
    ir0 = g.standard_normal((taps, S)) * 0.05
    x = torch.from_numpy(g.uniform(-1, 1, (S, n_hops * hop)).astype(np.float32)).cuda()
    dirs = [None if ir is None else torch.from_numpy(ir).cuda() for ir in irs]
    return ir0, x, dirs


def _loop(eng, x, dirs, period, hop):
    import torch

    n = x.shape[1] // hop
    out = torch.empty_like(x)
    for k in range(-(-n // period)):
        if dirs[k] is not None:
            eng.exchange_ir(dirs[k])
        sl = slice(k * period * hop, min(n, (k + 1) * period) * hop)
        eng.process_hops(x[:, sl], out=out[:, sl])
    return out


def _engines(monkeypatch, ir0, hop, warp_fft=False):
    a = T.TvolapEngine(T.partition(ir0, hop))
    a.set_tuning("wide", 2)
    a.set_tuning("wide_warp_fft", 1 if warp_fft else 0)
    b = T.TvolapEngine(T.partition(ir0, hop))
    b.set_tuning("wide", 0)
    return a, b


def _close(ya, yb, rel=2e-6):
    ya, yb = ya.cpu().numpy(), yb.cpu().numpy()
    return np.abs(ya - yb).max() <= rel * np.abs(yb).max()


@pytest.mark.parametrize("hop,S,taps,n_hops,period,none_at,pre", [
    (256, 5, 4096, 16 * 9, 16, (2,), 3),      # C2 geometry, odd start hop, one period without a switch
    (256, 3, 4096, 16 * 6 + 7, 16, (), 0),    # ragged final period (7 hops), first call
    (256, 3, 3000, 61, 10, (), 5),            # final period of 1 hop -> hop-blocked tail
    (256, 2, 4096, 100, 40, (1,), 2),         # 40-hop periods -> three tiles each
    (256, 2, 4096, 45, 3, (), 1),             # 3-hop periods (shortest tile)
    (128, 4, 2048, 150, 64, (), 4),           # N = 256, C1-like period
    (512, 2, 8192, 48, 8, (0,), 3),           # N = 1024, no switch at the first hop
    (32, 6, 1024, 90, 17, (), 2),             # N = 64, M = 16
    (64, 3, 8192, 70, 16, (), 1),             # N = 128, M = 64 (long history: ring wraps)
])
def test_wide_equals_exchange_loop(monkeypatch, hop, S, taps, n_hops, period, none_at, pre):
    ir0, x, dirs = _case(hop, S, taps, n_hops, period, none_at)
    a, b = _engines(monkeypatch, ir0, hop)
    if pre:
        a.process_hops(x[:, : pre * hop])
        b.process_hops(x[:, : pre * hop])
    ya = a.process_switching(x, dirs, period)
    yb = _loop(b, x, dirs, period, hop)
    a.synchronize()
    b.synchronize()
    assert a.wide_passes() >= 1 and b.wide_passes() == 0
    assert np.array_equal(ya.cpu().numpy(), yb.cpu().numpy())
    # state handed to the next calls: delay line, carry, history and the active set
    za, zb = a.process_hops(x[:, : 40 * hop]), b.process_hops(x[:, : 40 * hop])
    a.synchronize()
    b.synchronize()
    assert np.array_equal(za.cpu().numpy(), zb.cpu().numpy())
    assert a.op_counts() == b.op_counts()


@pytest.mark.parametrize("hop,S,taps,n_hops,period,none_at,pre", [
    (256, 5, 4096, 16 * 9, 16, (2,), 3),
    (256, 3, 3000, 61, 10, (), 5),
    (256, 2, 4096, 100, 40, (1,), 2),
    (128, 4, 2048, 150, 64, (), 4),
    (512, 2, 8192, 48, 8, (0,), 3),
    (32, 6, 1024, 90, 17, (), 2),
    (64, 3, 8192, 70, 16, (), 1),
])
def test_wide_warp_fft_matches_loop(monkeypatch, hop, S, taps, n_hops, period, none_at, pre):
    """Default mode (warp-per-frame K1/K5 transforms): the loop's outputs to fp32 rounding, and
    the state it hands on (delay line from the warp K1) keeps later calls within rounding."""
    ir0, x, dirs = _case(hop, S, taps, n_hops, period, none_at)
    a, b = _engines(monkeypatch, ir0, hop, warp_fft=True)
    if pre:
        a.process_hops(x[:, : pre * hop])
        b.process_hops(x[:, : pre * hop])
    ya = a.process_switching(x, dirs, period)
    yb = _loop(b, x, dirs, period, hop)
    a.synchronize()
    b.synchronize()
    assert a.wide_passes() >= 1
    assert _close(ya, yb)
    za, zb = a.process_hops(x[:, : 40 * hop]), b.process_hops(x[:, : 40 * hop])
    a.synchronize()
    b.synchronize()
    assert _close(za, zb)


def test_wide_chunked_pool(monkeypatch):
    """A pool budget of one set per chunk: every period is its own pass."""
    hop, S, taps, n, period = 256, 4, 4096, 16 * 7 + 5, 16
    ir0, x, dirs = _case(hop, S, taps, n, period, none_at=(3,))
    a, b = _engines(monkeypatch, ir0, hop)
    a.set_tuning("wide_pool_mb", 1)
    ya = a.process_switching(x, dirs, period)
    yb = _loop(b, x, dirs, period, hop)
    a.synchronize()
    b.synchronize()
    assert np.array_equal(ya.cpu().numpy(), yb.cpu().numpy())


@pytest.mark.parametrize("period,none_at", [(16, (0, 3)), (8, (2,)), (24, (1,))])
def test_wide_chunked_passes(monkeypatch, period, none_at):
    """A 1 MB extended-spectra budget: the call runs as several passes (fused K4 for periods of
    <= 16 hops, a partition_multi launch per pass otherwise); the set in effect crosses passes."""
    hop, S, taps, n = 256, 4, 4096, period * 9 + 5
    ir0, x, dirs = _case(hop, S, taps, n, period, none_at=none_at)
    a, b = _engines(monkeypatch, ir0, hop)
    a.set_tuning("wide_xe_mb", 1)
    ya = a.process_switching(x, dirs, period)
    yb = _loop(b, x, dirs, period, hop)
    a.synchronize()
    b.synchronize()
    assert a.wide_passes() > 1
    assert np.array_equal(ya.cpu().numpy(), yb.cpu().numpy())
    za, zb = a.process_hops(x[:, : 20 * hop]), b.process_hops(x[:, : 20 * hop])
    assert np.array_equal(za.cpu().numpy(), zb.cpu().numpy())


def test_wide_back_to_back_calls(monkeypatch):
    """Consecutive switching calls (the bench's step loop) hand the state over bit-exactly."""
    hop, S, taps, n, period = 256, 3, 4096, 64, 16
    ir0, x, dirs = _case(hop, S, taps, n, period)
    a, b = _engines(monkeypatch, ir0, hop)
    for _ in range(3):
        ya = a.process_switching(x, dirs, period)
        yb = _loop(b, x, dirs, period, hop)
        a.synchronize()
        b.synchronize()
        assert np.array_equal(ya.cpu().numpy(), yb.cpu().numpy())


def test_wide_matches_oracle(monkeypatch):
    hop, S, taps, n, period = 128, 2, 4096, 80, 16
    ir0, x, dirs = _case(hop, S, taps, n, period)
    eng_g = T.TvolapEngine(T.partition(ir0, hop))
    eng_g.set_tuning("wide", 2)
    y = eng_g.process_switching(x, dirs, period)
    eng_g.synchronize()
    y = y.cpu().numpy()
    xs = x.cpu().numpy().astype(np.float64)
    eng = O.Engine(O.partition(ir0.astype(np.float32).astype(np.float64), hop))
    ref = []
    for h in range(n):
        if h % period == 0 and dirs[h // period] is not None:
            eng.exchange_filter(O.partition(dirs[h // period].cpu().numpy().T.astype(np.float64), hop,
                                            eng.partition_count()))
        ref.append(eng.process(xs[:, h * hop:(h + 1) * hop].T))
    ref = np.concatenate(ref).T
    err = np.max(np.abs(y - ref)) / np.max(np.abs(ref))
    assert err <= 1e-4, err  # north-star tolerance (fp32 vs the fp64 reference algorithm)


@pytest.mark.parametrize("first_switch", [False, True])
def test_wide_after_staged_exchange(monkeypatch, first_switch):
    """A filter staged with exchange_filter before the call is latched at its first hop (irs[0] is
    None), or superseded when irs[0] names a set (last staged wins, engine.cpp:47)."""
    hop, S, taps, n, period = 256, 3, 4096, 16 * 5, 16
    ir0, x, dirs = _case(hop, S, taps, n, period, none_at=() if first_switch else (0,))
    import torch

    staged = torch.from_numpy(np.random.default_rng(9).standard_normal((S, taps)).astype(np.float32) * 0.05).cuda()
    a, b = _engines(monkeypatch, ir0, hop)
    a.process_hops(x[:, : 2 * hop])
    b.process_hops(x[:, : 2 * hop])
    a.exchange_ir(staged)
    b.exchange_ir(staged)
    ya = a.process_switching(x, dirs, period)
    yb = _loop(b, x, dirs, period, hop)
    a.synchronize()
    b.synchronize()
    assert a.wide_passes() >= 1
    assert np.array_equal(ya.cpu().numpy(), yb.cpu().numpy())


def _bank_engines(monkeypatch, bank, hop, S):
    """a: piecewise time-parallel passes forced; b: the hop-blocked launch only (no pass of either
    kind; the per-hop bank pass is tested in test_gpu_bank_pass.py)."""
    a = T.TvolapBankEngine(bank, hop, S)
    a.set_tuning("wide", 2)
    a.set_tuning("bank_pass", 0)
    b = T.TvolapBankEngine(bank, hop, S)
    b.set_tuning("wide", 0)
    b.set_tuning("bank_pass", 0)
    return a, b


@pytest.mark.parametrize("hop,S,taps,n_hops,seg", [
    (128, 1, 4096, 200, 64),   # C1 shape: one lane, two entries alternating every 64 hops
    (256, 3, 4096, 120, 20),   # several lanes changing together every 20 hops
    (64, 2, 2048, 90, 7),      # short segments (7-hop tiles), N = 128
])
def test_wide_bank_schedule_equals_blocked(monkeypatch, hop, S, taps, n_hops, seg):
    """Bank engines on device buffers with a piecewise-constant schedule: time-parallel passes
    (Stockham transforms) == the hop-blocked launch bit for bit, state included."""
    import torch

    g = np.random.default_rng(3)
    n_bank = 3
    bank = (g.standard_normal((n_bank, 1, taps)) * 0.05).astype(np.float32)
    x = torch.from_numpy(g.uniform(-1, 1, (S, n_hops * hop)).astype(np.float32)).cuda()
    h = np.arange(n_hops)
    sched = np.stack([((h // seg) + s) % n_bank for s in range(S)], 1).astype(np.int32)
    sched_d = torch.from_numpy(sched).cuda()
    a, b = _bank_engines(monkeypatch, bank, hop, S)
    a.process_hops(x[:, : 3 * hop], schedule=sched_d[:3])  # (short call: hop-blocked in both)
    b.process_hops(x[:, : 3 * hop], schedule=sched_d[:3])
    ya = a.process_hops(x, schedule=sched_d)
    yb = b.process_hops(x, schedule=sched_d)
    a.synchronize()
    b.synchronize()
    assert a.wide_passes() >= 1 and b.wide_passes() == 0
    assert np.array_equal(ya.cpu().numpy(), yb.cpu().numpy())
    za = a.process_hops(x[:, : 20 * hop], schedule=sched_d[:20])
    zb = b.process_hops(x[:, : 20 * hop], schedule=sched_d[:20])
    a.synchronize()
    b.synchronize()
    assert np.array_equal(za.cpu().numpy(), zb.cpu().numpy())
    # the schedule's last row stays latched for later process() calls (no schedule)
    xs = x.cpu().numpy()
    for k in range(3):
        blk = np.ascontiguousarray(xs[:, k * hop:(k + 1) * hop].T)
        assert np.array_equal(a.process(blk), b.process(blk))
    assert a.op_counts() == b.op_counts()


def test_wide_bank_pinned_host_pipeline(monkeypatch):
    """Pinned host buffers + host schedule (the C1 e2e path): each pipeline chunk runs as a
    time-parallel pass; equal bit for bit to the device call on the hop-blocked launch."""
    import torch

    g = np.random.default_rng(5)
    hop, S, taps, n = 128, 1, 8192, 300
    bank = (g.standard_normal((2, 1, taps)) * 0.05).astype(np.float32)
    xs = g.uniform(-1, 1, (S, n * hop)).astype(np.float32)
    sched = ((np.arange(n) // 64) % 2).astype(np.int32)[:, None]
    a, b = _bank_engines(monkeypatch, bank, hop, S)
    xh = torch.from_numpy(xs).pin_memory()
    yh = torch.empty(xh.shape, dtype=torch.float32).pin_memory()
    a.process_hops(xh, out=yh, schedule=sched)
    a.synchronize()
    yd = b.process_hops(torch.from_numpy(xs).cuda(), schedule=torch.from_numpy(sched).cuda())
    b.synchronize()
    assert a.wide_passes() >= 1
    assert np.array_equal(yh.numpy(), yd.cpu().numpy())


def test_wide_bank_random_schedule_stays_blocked(monkeypatch):
    """A schedule that changes every hop (C3/C5) has no >= 3-hop segments: no piecewise pass;
    with the bank pass switched off the call stays on the hop-blocked kernel."""
    import torch

    g = np.random.default_rng(4)
    bank = (g.standard_normal((4, 1, 2048)) * 0.05).astype(np.float32)
    a, _ = _bank_engines(monkeypatch, bank, 128, 2)
    a.set_tuning("bank_pass", 0)
    x = torch.from_numpy(g.uniform(-1, 1, (2, 64 * 128)).astype(np.float32)).cuda()
    sched = torch.from_numpy(g.integers(0, 4, (64, 2)).astype(np.int32)).cuda()
    a.process_hops(x, schedule=sched)
    a.synchronize()
    assert a.wide_passes() == 0


@pytest.mark.parametrize("hop,S,taps,n_hops", [(256, 2, 4096, 200), (128, 1, 8192, 97), (512, 3, 16384, 64)])
def test_wide_set_process_hops_equals_one_hop(monkeypatch, hop, S, taps, n_hops):
    """Filter-set engines: a device-resident process_hops call runs as a time-parallel pass and
    equals hop-by-hop process() bit for bit (and the state it leaves behind)."""
    import torch

    g = np.random.default_rng(6)
    ir = g.standard_normal((taps, S)) * 0.05
    a = T.TvolapEngine(T.partition(ir, hop))
    a.set_tuning("wide", 2)
    b = T.TvolapEngine(T.partition(ir, hop))
    xs = g.uniform(-1, 1, (S, (n_hops + 5) * hop)).astype(np.float32)
    ya = a.process_hops(torch.from_numpy(np.ascontiguousarray(xs[:, : n_hops * hop])).cuda())
    a.synchronize()
    assert a.wide_passes() >= 1
    yb = np.concatenate([b.process(np.ascontiguousarray(xs[:, k * hop:(k + 1) * hop].T)).T for k in range(n_hops)], 1)
    assert np.array_equal(ya.cpu().numpy(), yb)
    for k in range(n_hops, n_hops + 5):  # the carry, history and delay line handed on
        blk = np.ascontiguousarray(xs[:, k * hop:(k + 1) * hop].T)
        assert np.array_equal(a.process(blk), b.process(blk))
