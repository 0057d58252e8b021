"""Bank pass (tvolap_wide.cu bank_mac_kernel / bank_k5_kernel): bank engines whose per-hop schedule
changes every hop (C3, C5) on device-resident hops. Checked against the reference engine (oracle,
the reference's own sources where oracle/_ref is present), against the hop-blocked kernel to fp32
rounding, and for invariance (bit for bit) under pass splitting and the pinned-host pipeline."""
import numpy as np
import pytest

from paper_2310_00319_b200 import tvolap as T
from parity import TOL, best_oracle

import oracle as O

pytestmark = pytest.mark.gpu


def _case(hop, S, ears, n_bank, taps, n, seed):
    g = np.random.default_rng(seed)
    bank = (g.standard_normal((n_bank, ears, taps)) * np.exp(-np.arange(taps) / (taps / 4))).astype(np.float32)
    x = g.uniform(-1, 1, (S, n * hop)).astype(np.float32)
    sched = g.integers(0, n_bank, (n, S)).astype(np.int32)
    return bank, x, sched


def _oracle(bank, x, sched, hop, M):
    S, ears = x.shape[0], bank.shape[1]
    n = sched.shape[0]
    with O.using(best_oracle()):
        _, y = O.run_workload(hop, M, S, ears, n, x.astype(np.float64), 1, bank_ir=bank.astype(np.float64),
                              schedule=sched, threads=8)
    return y


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("hop,S,ears,n_bank,taps,n,pre", [
    (32, 6, 1, 9, 4096, 300, 0),     # C5 shape (N = 64, tiles of <= 64 hops), ring wrapped (M = 64)
    (32, 3, 1, 5, 1500, 97, 5),      # ragged tiles, odd start hop after a short call
    (128, 4, 2, 6, 4096, 120, 3),    # C3 shape (N = 256, two ears share the source spectrum)
    (64, 2, 1, 4, 2048, 70, 0),      # N = 128
    (256, 2, 2, 3, 3000, 66, 1),     # N = 512, two ears
])
def test_bank_pass_matches_reference(hop, S, ears, n_bank, taps, n, pre):
    bank, x, sched = _case(hop, S, ears, n_bank, taps, n + pre, 11 + hop)
    e = T.TvolapBankEngine(bank, hop, S)
    M = e.partition_count()
    xd, sd = _dev(x), _dev(sched)
    parts = []
    if pre:  # a few hops on the hop-blocked / one-hop kernels first: the pass starts mid-stream
        parts.append(e.process_hops(xd[:, : pre * hop], schedule=sd[:pre]))
    p0 = e.wide_passes()
    parts.append(e.process_hops(xd[:, pre * hop:], schedule=sd[pre:]))
    e.synchronize()
    assert e.wide_passes() > p0, "the per-hop schedule should run as a bank pass"
    y = np.concatenate([p.cpu().numpy() for p in parts], 1)
    ref = _oracle(bank, x, sched, hop, M)
    err = np.abs(y - ref).max() / np.abs(ref).max()
    assert err <= TOL, err
    # the state it hands on: more hops on the streaming kernel continue the same stream
    xb = np.random.default_rng(2).uniform(-1, 1, (S, 6 * hop)).astype(np.float32)
    sb = np.random.default_rng(3).integers(0, n_bank, (6, S)).astype(np.int32)
    tail = []
    for h in range(6):
        e.select_bank(sb[h])
        tail.append(e.process(np.ascontiguousarray(xb[:, h * hop:(h + 1) * hop].T)).T)
    ref2 = _oracle(bank, np.concatenate([x, xb], 1), np.concatenate([sched, sb]), hop, M)
    got = np.concatenate(tail, 1)
    err2 = np.abs(got - ref2[:, -6 * hop:]).max() / np.abs(ref2).max()
    assert err2 <= TOL, err2


@pytest.mark.parametrize("hop,ears", [(32, 1), (128, 2)])
def test_bank_pass_vs_hop_blocked_kernel(hop, ears):
    """Same sums in a different partition grouping / transform factorisation: fp32 rounding apart."""
    S, n_bank, taps, n = 5, 7, 3000, 80
    bank, x, sched = _case(hop, S, ears, n_bank, taps, n, 21)
    a = T.TvolapBankEngine(bank, hop, S)
    b = T.TvolapBankEngine(bank, hop, S)
    b.set_tuning("bank_pass", 0)
    ya = a.process_hops(_dev(x), schedule=_dev(sched)).cpu().numpy()
    yb = b.process_hops(_dev(x), schedule=_dev(sched)).cpu().numpy()
    assert a.wide_passes() >= 1 and b.wide_passes() == 0
    assert np.abs(ya - yb).max() <= 2e-6 * np.abs(yb).max()


@pytest.mark.parametrize("hop,ears", [(32, 1), (128, 2)])
def test_bank_pass_split_and_pinned_are_bit_identical(hop, ears):
    """Pass boundaries (passes of 2J hops) and the pinned-host pipeline's chunks change
    nothing: every output is the same per-output sum, transform and overlap-add order."""
    import torch

    S, n_bank, taps, n = 4, 6, 2500, 700
    bank, x, sched = _case(hop, S, ears, n_bank, taps, n, 31)
    a = T.TvolapBankEngine(bank, hop, S)
    ya = a.process_hops(_dev(x), schedule=_dev(sched)).cpu().numpy()
    b = T.TvolapBankEngine(bank, hop, S)
    b.set_tuning("bank_pass_hops", 1)  # -> 2J hops per pass
    yb = b.process_hops(_dev(x), schedule=_dev(sched)).cpu().numpy()
    assert b.wide_passes() > a.wide_passes() >= 1
    assert np.array_equal(ya, yb)
    c = T.TvolapBankEngine(bank, hop, S)
    c.set_tuning("pipe_log2", 10)  # small pinned chunks (8M hops each: several chunks, each a bank pass)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty((S * ears, n * hop), dtype=torch.float32).pin_memory()
    c.process_hops(xh, out=yh, schedule=sched)
    c.synchronize()
    assert c.wide_passes() >= 2
    assert np.array_equal(ya, yh.numpy())
    # and all three leave the same state behind
    xs = np.ascontiguousarray(x[:, : hop].T)
    for eng in (a, b, c):
        eng.select_bank(sched[0])
    za, zb, zc = a.process(xs), b.process(xs), c.process(xs)
    assert np.array_equal(za, zb) and np.array_equal(za, zc)


def test_bank_pass_tuning_switch():
    assert "bank_pass" in T.tuning_keys()
    bank, x, sched = _case(32, 2, 1, 4, 1000, 70, 41)
    e = T.TvolapBankEngine(bank, 32, 2)
    assert e.get_tuning("bank_pass") == 1
    e.set_tuning("bank_pass", 0)
    e.process_hops(_dev(x), schedule=_dev(sched))
    e.synchronize()
    assert e.wide_passes() == 0
    with pytest.raises(T.InvalidInputError):
        e.set_tuning("bank_pass", 7)
    with pytest.raises(T.InvalidInputError):
        e.set_tuning("no_such_knob", 1)


def test_bank_pass_tile_geometry_knobs():
    """Tile size (bank_pass_jh: 16 / 32 / 64-hop tiles) and tiles per MAC CTA (bank_pass_tpc: how
    many consecutive tiles a CTA walks so its Xe window stays in L1) only regroup the work: the
    tpc variants are bit-identical, every tile size matches the reference."""
    hop, S, n_bank, taps, n = 32, 5, 7, 4096, 333
    bank, x, sched = _case(hop, S, 1, n_bank, taps, n, 51)
    ref = None
    outs = {}
    for jh in (8, 16, 32):
        for tpc in (1, 2, 0):
            e = T.TvolapBankEngine(bank, hop, S)
            e.set_tuning("bank_pass_jh", jh)
            e.set_tuning("bank_pass_tpc", tpc)
            assert e.get_tuning("bank_pass_jh") == jh and e.get_tuning("bank_pass_tpc") == tpc
            y = e.process_hops(_dev(x), schedule=_dev(sched)).cpu().numpy()
            assert e.wide_passes() >= 1
            outs[jh, tpc] = y
            if ref is None:
                ref = _oracle(bank, x, sched, hop, e.partition_count())
        assert np.array_equal(outs[jh, 1], outs[jh, 2]) and np.array_equal(outs[jh, 1], outs[jh, 0])
        err = np.abs(outs[jh, 0] - ref).max() / np.abs(ref).max()
        assert err <= TOL, (jh, err)
    assert np.abs(outs[8, 0] - outs[32, 0]).max() <= 2e-6 * np.abs(ref).max()
    # two-ear engines (C3 geometry): 16- or 32-hop tiles; the tiles-per-CTA walk applies to them too
    bank2, x2, sched2 = _case(128, 3, 2, 5, 3000, 90, 52)
    ys = {}
    for jh in (8, 16):
        for tpc in (1, 0):
            e = T.TvolapBankEngine(bank2, 128, 3)
            e.set_tuning("bank_pass_jh", jh)
            e.set_tuning("bank_pass_tpc", tpc)
            ys[jh, tpc] = e.process_hops(_dev(x2), schedule=_dev(sched2)).cpu().numpy()
        assert np.array_equal(ys[jh, 0], ys[jh, 1])
    ref2 = _oracle(bank2, x2, sched2, 128, e.partition_count())
    for jh in (8, 16):
        assert np.abs(ys[jh, 0] - ref2).max() <= TOL * np.abs(ref2).max()
    assert np.abs(ys[8, 0] - ys[16, 0]).max() <= 2e-6 * np.abs(ref2).max()
