"""Pin the CPU oracle to the reference's own known-answer and property tests.

The reference ships no golden vectors; its spectral, partition
and engine suites are brute-force property/KAT tests. Each test below restates
one of them (file:line cited) with the same tolerances, against the fp64
oracle (oracle/tvolap_oracle.cpp). Inputs use numpy's seeded generator instead
of libstdc++'s uniform_real_distribution (whose values are library-specific).
"""
import numpy as np
import pytest

import oracle as O


def rnd(n, seed, cols=None):
    g = np.random.default_rng(seed)
    return g.uniform(-1, 1, n if cols is None else (n, cols))


# numpy brute-force references (proj/tests/oracles.hpp:15-43)
def naive_dft(x):
    n = x.size
    k = np.arange(n)
    return (x[None, :] * np.exp(-2j * np.pi * np.outer(k, k) / n)).sum(1)


def circular_conv(x, h):
    n = x.size
    return np.array([sum(x[i] * h[(k - i) % n] for i in range(n)) for k in range(n)])


def linear_conv(x, h):
    return np.convolve(x, h)


def delta_ir(gain, length):
    h = np.zeros(length)
    h[0] = gain
    return h


# ------------------------------------------------------------ spectral (test_spectral.cpp)
def test_impulse_flat_spectrum():  # test_spectral.cpp:32-42
    x = np.zeros(8)
    x[0] = 1
    s = O.forward_real(x)
    assert s.size == 5
    assert np.allclose(s.real, 1.0, rtol=1e-14) and np.abs(s.imag).max() < 1e-15


def test_constant_is_dc_only():  # test_spectral.cpp:44-49
    s = O.forward_real(np.ones(8))
    assert s[0] == 8.0
    assert np.abs(s[1:]).max() < 1e-14


@pytest.mark.parametrize("n", [8, 16, 64, 256, 1024])
def test_forward_matches_naive_dft(n):  # test_spectral.cpp:51-62
    x = rnd(n, 100 + n)
    s = O.forward_real(x)
    assert s.size == n // 2 + 1
    assert np.abs(s - naive_dft(x)[: n // 2 + 1]).max() < 1e-12 * max(1.0, n / 64.0)


def test_roundtrip_all_sizes():  # test_spectral.cpp:64-71
    n = 8
    while n <= 8192:
        x = rnd(n, 200 + n)
        assert np.abs(O.inverse_real(O.forward_real(x)) - x).max() < 1e-12
        n *= 2


def test_roundtrip_impulse_and_zero():  # test_spectral.cpp:73-82
    x = np.zeros(8)
    x[0] = 1
    assert np.abs(O.inverse_real(O.forward_real(x)) - x).max() < 1e-15
    z = O.inverse_real(np.zeros(33, complex), 64)
    assert z.size == 64 and np.abs(z).max() == 0.0


def test_forward_linear():  # test_spectral.cpp:84-94
    x, y = rnd(512, 1), rnd(512, 2)
    a, b = 0.7, -1.9
    lhs = O.forward_real(a * x + b * y)
    assert np.abs(lhs - (a * O.forward_real(x) + b * O.forward_real(y))).max() < 1e-12


@pytest.mark.parametrize("n", [8, 16, 32])
def test_product_is_circular_conv(n):  # test_spectral.cpp:96-107
    x, h = rnd(n, 300 + n), rnd(n, 400 + n)
    prod = O.mac(np.zeros(n // 2 + 1, complex), O.forward_real(x), O.forward_real(h))
    assert np.abs(O.inverse_real(prod) - circular_conv(x, h)).max() < 1e-10


def test_mac_matches_scalar_complex():  # test_spectral.cpp:109-127 (exact)
    g = np.random.default_rng(5)
    f = lambda: g.uniform(-1, 1, 33) + 1j * g.uniform(-1, 1, 33)  # noqa: E731
    acc, a, b = f(), f(), f()
    out = O.mac(acc, a, b)
    want = acc + (a.real * b.real - a.imag * b.imag) + 1j * (a.real * b.imag + a.imag * b.real)
    assert np.array_equal(out, want)
    assert acc[3] != out[3]


def test_mac_identities():  # test_spectral.cpp:129-141
    s = O.forward_real(rnd(32, 6))
    flat = np.ones(17, complex)
    assert np.abs(O.mac(np.zeros(17, complex), flat, s) - s).max() == 0.0
    assert np.abs(O.mac(s, np.zeros(17, complex), flat) - s).max() == 0.0


def test_spectral_validation():  # test_spectral.cpp:143-161
    for n in (4, 12, 0):
        with pytest.raises(O.OracleError) as e:
            O.forward_real(np.zeros(n))
        assert e.value.code == 1  # InvalidSizeError
    bad = np.zeros(9, complex)
    bad[0] = 1e-3j
    with pytest.raises(O.OracleError) as e:
        O.inverse_real(bad, 16)
    assert e.value.code == 5  # InvalidSpectrumError
    bad = np.zeros(9, complex)
    bad[8] = 1e-3j
    with pytest.raises(O.OracleError) as e:
        O.inverse_real(bad, 16)
    assert e.value.code == 5
    with pytest.raises(O.OracleError) as e:
        O.inverse_real(np.zeros(4, complex), 16)
    assert e.value.code == 1
    with pytest.raises(O.OracleError) as e:
        O.mac(np.zeros(9, complex), np.zeros(9, complex), np.zeros(17, complex))
    assert e.value.code == 1


# ------------------------------------------------------------ partition (test_partition.cpp)
def test_window_endpoints_peak_overlap():  # test_partition.cpp:25-34
    w = O.hann_window(256)
    assert w.size == 512 and w[0] == 0.0 and w[256] == 2.0
    assert np.allclose(w[:256] + w[256:], 2.0, rtol=1e-15)


@pytest.mark.parametrize("hop", [2, 16, 128])
def test_window_cola(hop):  # test_partition.cpp:36-42
    w = O.hann_window(hop)
    assert np.abs(w[:hop] + w[hop:] - 2.0).max() < 1e-15


def test_window_rejects_degenerate():  # test_partition.cpp:44-47
    for hop in (1, 0):
        with pytest.raises(O.OracleError):
            O.hann_window(hop)


def test_partition_counts():  # test_partition.cpp:49-55
    assert O.partition(rnd(2048, 1), 256).partition_count == 4
    assert O.partition(rnd(1536, 2, 2), 256).partition_count == 3
    assert O.partition(rnd(1, 3), 256).partition_count == 1
    assert O.partition(rnd(1000, 4), 256).partition_count == 2
    assert O.partition(rnd(513, 5), 256).partition_count == 2


def test_unit_impulse_partitions_flat():  # test_partition.cpp:57-69
    s = O.partition(np.ones(1), 256)
    assert s.partition_count == 1 and s.transform_length() == 1024 and s.normalization_gain == 0.5
    sp = s.spectra()[0, 0]
    assert np.allclose(sp.real, 1.0, rtol=1e-13) and np.abs(sp.imag).max() < 1e-13


def test_reassemble_inverts():  # test_partition.cpp:71-78
    ir = rnd(2048, 10, 2)
    back = O.partition(ir, 256).reassemble()
    assert back.shape == (2048, 2)
    assert np.abs(back - ir).max() < 1e-12


def test_odd_length_tail_padding():  # test_partition.cpp:80-89
    ir = rnd(1000, 11)
    s = O.partition(ir, 256)
    assert s.source_length == 1000 and s.padded_length() == 1024
    back = s.reassemble()[:, 0]
    assert np.abs(back[:1000] - ir).max() < 1e-12 and np.abs(back[1000:]).max() < 1e-12


def test_partition_linear():  # test_partition.cpp:100-112
    a, b = 1.25, -0.5
    i1, i2 = rnd(700, 12), rnd(700, 13)
    s1, s2, sm = (O.partition(v, 128).spectra() for v in (i1, i2, a * i1 + b * i2))
    assert np.abs(sm - (a * s1 + b * s2)).max() < 1e-12


def test_min_partitions_forces_zero_tail():  # test_partition.cpp:114-122
    s = O.partition(rnd(512, 14), 256, 4)
    assert s.partition_count == 4
    assert np.abs(s.spectra()[0, 1:]).max() == 0.0


def test_partition_validation():  # test_partition.cpp:124-130
    with pytest.raises(O.OracleError) as e:
        O.partition(np.zeros((0, 1)), 256)
    assert e.value.code == 2
    for hop in (0, 24, 1):
        with pytest.raises(O.OracleError) as e:
            O.partition(rnd(64, 15), hop)
        assert e.value.code == 1


# ------------------------------------------------------------ engine (test_engine.cpp)
def test_engine_geometry():  # test_engine.cpp:42-58
    one = O.Engine(O.partition(delta_ir(1, 1), 256))
    assert (one.partition_count(), one.latency(), one.switching_latency(), one.delay_line_depth()) == (1, 512, 256, 1)
    four = O.Engine(O.partition(delta_ir(1, 2048), 256))
    assert (four.partition_count(), four.delay_line_depth(), four.hop(), four.channels()) == (4, 7, 256, 1)
    big = O.Engine(O.partition(delta_ir(1, 32768), 512))
    assert big.partition_count() == 32 and big.switching_latency() == 512


def test_zero_stays_zero_after_reset():  # test_engine.cpp:60-69
    eng = O.Engine(O.partition(delta_ir(1, 1024), 128))
    z = np.zeros((128, 1))
    for _ in range(5):
        assert np.abs(eng.process(z)).max() == 0.0
    eng.process(rnd(128, 1, 1))
    eng.reset()
    for _ in range(5):
        assert np.abs(eng.process(z)).max() == 0.0


def test_identity_passthrough():  # test_engine.cpp:71-77
    eng = O.Engine(O.partition(delta_ir(1, 1), 16))
    x = rnd(128, 2, 1)
    assert np.abs(O.stream_through(eng, x, 128) - x).max() < 1e-12


@pytest.mark.parametrize("n_ir", [256, 512, 1024])
def test_fixed_filter_matches_linear_conv(n_ir):  # test_engine.cpp:79-89
    h, x = rnd(n_ir, 10 + n_ir), rnd(4 * n_ir, 20 + n_ir)
    eng = O.Engine(O.partition(h, 128))
    y = O.stream_through(eng, x, x.size + n_ir - 1)[:, 0]
    assert np.abs(y - linear_conv(x, h)).max() < 1e-9


def test_channels_independent():  # test_engine.cpp:91-102
    ir, x = rnd(256, 30, 2), rnd(1024, 31, 2)
    eng = O.Engine(O.partition(ir, 64))
    assert eng.channels() == 2
    y = O.stream_through(eng, x, 1024 + 255)
    for c in range(2):
        assert np.abs(y[:, c] - linear_conv(x[:, c], ir[:, c])).max() < 1e-9


def test_engine_linear():  # test_engine.cpp:104-116
    s = O.partition(rnd(512, 40), 64)
    x1, x2 = rnd(512, 41), rnd(512, 42)
    a, b = 0.8, -2.5
    y1 = O.stream_through(O.Engine(s), x1, 900)
    y2 = O.stream_through(O.Engine(s), x2, 900)
    ym = O.stream_through(O.Engine(s), a * x1 + b * x2, 900)
    assert np.abs(ym - (a * y1 + b * y2)).max() < 1e-10


def test_constant_op_counts_through_exchange():  # test_engine.cpp:118-139, acceptance.cpp:154-174
    a, b = O.partition(rnd(1024, 50), 128), O.partition(rnd(1024, 51), 128)
    eng = O.Engine(a)
    m = eng.partition_count()
    for i in range(12):
        if i == 6:
            eng.exchange_filter(b)
        eng.process(np.ones((128, 1)))
        assert eng.op_counts() == (i + 1, i + 1, (i + 1) * m)


def test_exchange_identical_is_bit_identical():  # test_engine.cpp:141-157
    s = O.partition(rnd(512, 60), 64)
    x = rnd(1024, 61)
    plain, exch = O.Engine(s), O.Engine(s)
    for i in range(16):
        chunk = x[i * 64:(i + 1) * 64, None]
        y1 = plain.process(chunk)
        if i == 7:
            exch.exchange_filter(s)
        assert np.array_equal(y1, exch.process(chunk))


def half_cosine_stream(make_engine, process, exchange, stream_delay):
    hop, calls, switch_call = 256, 24, 12
    pos, neg = delta_ir(1, 2048), delta_ir(-1, 2048)
    eng = make_engine(pos, hop)
    stream = []
    for i in range(calls):
        if i == switch_call:
            exchange(eng, neg, hop)
        stream.append(process(eng, np.ones((hop, 1))))
    out = np.concatenate(stream)[stream_delay:, 0]
    return out, (switch_call - 1) * hop, hop


def test_polarity_flip_half_cosine():  # test_engine.cpp:159-188
    out, boundary, hop = half_cosine_stream(lambda h, L: O.Engine(O.partition(h, L)), lambda e, x: e.process(x),
                                            lambda e, h, L: e.exchange_filter(O.partition(h, L)), 256)
    w = O.hann_window(hop)
    assert np.allclose(out[2 * hop:boundary], 1.0, rtol=1e-9)
    expected = 0.5 * w[hop:] - 0.5 * w[:hop]
    assert np.allclose(out[boundary:boundary + hop], expected, rtol=1e-9, atol=1e-12)
    assert np.allclose(out[boundary + hop:], -1.0, rtol=1e-9)
    assert abs(out[boundary + hop - 1] + 1.0) > 1e-9


def test_shorter_ir_via_min_partitions():  # test_engine.cpp:190-201
    long_ir, short_ir = rnd(512, 70), rnd(100, 71)
    eng = O.Engine(O.partition(long_ir, 64))
    assert eng.partition_count() == 4
    eng.exchange_filter(O.partition(short_ir, 64, eng.partition_count()))
    x = rnd(2048, 72)
    y = O.stream_through(eng, x, x.size + 99)[:, 0]
    assert np.abs(y - linear_conv(x, short_ir)).max() < 1e-9


def test_framing_and_compatibility_enforced():  # test_engine.cpp:203-216
    eng = O.Engine(O.partition(delta_ir(1, 512), 128))
    with pytest.raises(O.OracleError) as e:
        eng.process(np.zeros((127, 1)))
    assert e.value.code == 1
    with pytest.raises(O.OracleError) as e:
        eng.process(np.zeros((128, 2)))
    assert e.value.code == 2
    for bad in (O.partition(delta_ir(1, 512), 64), O.partition(delta_ir(1, 2048), 128),
                O.partition(np.zeros((512, 2)) + np.eye(512, 2), 128)):
        with pytest.raises(O.OracleError) as e:
            eng.exchange_filter(bad)
        assert e.value.code == 4
    with pytest.raises(O.OracleError) as e:
        O.Engine(None)
    assert e.value.code == 3


def test_reset_keeps_staged_filter():  # test_engine.cpp:218-232
    eng = O.Engine(O.partition(delta_ir(1, 256), 64))
    eng.process(rnd(64, 80, 1))
    eng.exchange_filter(O.partition(delta_ir(-1, 256), 64))
    eng.reset()
    for _ in range(8):
        last = eng.process(np.ones((64, 1)))
    assert last[63, 0] == pytest.approx(-1.0, rel=1e-10)


def test_acceptance_crit2_vs_direct_convolve():  # acceptance.cpp:92-122 (tvolap leg, 6 of 20 pairs)
    for i in range(6):
        n_ir = (512, 1024, 2048)[i % 3]
        hop = (128, 256)[i % 2]
        ir, x = rnd(n_ir, 1000 + i), rnd(8192, 2000 + i)
        ref = O.direct_convolve(x, ir)
        y = O.stream_through(O.Engine(O.partition(ir, hop)), x, ref.size)[:, 0]
        assert np.abs(y - ref).max() < 1e-9


def test_direct_convolve_matches_numpy():  # reference.cpp:10-32
    x, h = rnd(300, 90), rnd(77, 91)
    assert np.abs(O.direct_convolve(x, h) - np.convolve(x, h)).max() < 1e-12


def test_closed_form_overlap_add():  # SURVEY.md Appendix A (engine.cpp:97-102 restated)
    L, M = 16, 3
    ir, x = rnd(2 * L * M, 7), rnd(12 * L, 8)
    s = O.partition(ir, L)
    eng = O.Engine(s)
    H = s.spectra()[0]
    w = O.hann_window(L)
    xs = np.concatenate([np.zeros(L), x])
    X, Y, out = [], [], []
    for l in range(12):
        blk = np.zeros(4 * L)
        blk[:2 * L] = xs[l * L:(l + 2) * L] * w
        X.append(np.fft.rfft(blk))
        acc = sum(H[m] * (X[l - 2 * m] if l - 2 * m >= 0 else 0) for m in range(M))
        Y.append(np.fft.irfft(acc, 4 * L))
        o = Y[l][:L].copy()
        for d in (1, 2, 3):
            if l - d >= 0:
                o += Y[l - d][d * L:(d + 1) * L]
        out.append(0.5 * o)
        assert np.abs(eng.process(x[l * L:(l + 1) * L, None])[:, 0] - out[-1]).max() < 1e-12


def test_workload_driver_matches_engine():
    """orc_run_workload (threaded drive loop) == one engine per lane driven by hand."""
    L, M, S = 16, 4, 3
    n_hops, period = 40, 8
    x = rnd(n_hops * L, 5, S).T.copy()
    irs = rnd(S * 5 * 2 * L * M, 6).reshape(5, S, 1, 2 * L * M)
    secs, y = O.run_workload(L, 1, S, 1, n_hops, x, 0, fresh_ir=irs, period=period, threads=2)
    for s in range(S):
        eng = O.Engine(O.partition(irs[0, s, 0], L))
        for h in range(n_hops):
            if h and h % period == 0:
                eng.exchange_filter(O.partition(irs[h // period, s, 0], L, M))
            yy = eng.process(x[s, h * L:(h + 1) * L, None])[:, 0]
            assert np.array_equal(yy, y[s, h * L:(h + 1) * L])
    # bank mode with two ears sharing the input
    bank = rnd(4 * 2 * 2 * L * M, 9).reshape(4, 2, 2 * L * M)
    sched = np.random.default_rng(3).integers(0, 4, (n_hops, S)).astype(np.int32)
    _, yb = O.run_workload(L, 1, S, 2, n_hops, x, 1, bank_ir=bank, schedule=sched, threads=3)
    for s in range(S):
        eng = O.Engine(O.partition(bank[sched[0, s]].T, L))
        cur = sched[0, s]
        for h in range(n_hops):
            if h and sched[h, s] != cur:
                eng.exchange_filter(O.partition(bank[sched[h, s]].T, L))
                cur = sched[h, s]
            seg = np.repeat(x[s, h * L:(h + 1) * L, None], 2, axis=1)
            yy = eng.process(seg)
            assert np.array_equal(yy[:, 0], yb[2 * s, h * L:(h + 1) * L])
            assert np.array_equal(yy[:, 1], yb[2 * s + 1, h * L:(h + 1) * L])
