"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle and the
reference's known answers. Mirrors proj/tests/test_spectral.cpp,
test_partition.cpp and test_engine.cpp at fp32 tolerances."""
import numpy as np
import pytest

import oracle as O
from paper_2310_00319_b200 import tvolap as T

pytestmark = pytest.mark.gpu


def rnd(n, seed, cols=None):
    g = np.random.default_rng(seed)
    return g.uniform(-1, 1, n if cols is None else (n, cols))


def delta_ir(gain, length):
    h = np.zeros(length)
    h[0] = gain
    return h


def stream_through(eng, x, n_out):
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    hop = eng.hop()
    total = n_out + eng.stream_delay()
    calls = -(-total // hop)
    padded = np.zeros((calls * hop, x.shape[1]))
    padded[: x.shape[0]] = x
    out = np.concatenate([eng.process(padded[i * hop:(i + 1) * hop]) for i in range(calls)])
    return out[eng.stream_delay(): eng.stream_delay() + n_out].astype(np.float64)


# ------------------------------------------------------------ spectral
def test_forward_real_vs_oracle_and_dft():  # test_spectral.cpp:32-62
    x = np.zeros(8)
    x[0] = 1
    s = T.forward_real(x)
    assert np.allclose(s, 1.0, atol=1e-6)
    assert abs(T.forward_real(np.ones(8))[0] - 8.0) < 1e-6
    for n in (8, 16, 64, 256, 1024, 2048, 4096):
        x = rnd(n, 100 + n).astype(np.float32)
        got = T.forward_real(x)
        ref = O.forward_real(x.astype(np.float64))
        assert np.abs(got - ref).max() < 2e-6 * np.sqrt(n) * max(1.0, np.log2(n) / 4)
        assert got[0].imag == 0 and got[-1].imag == 0


def test_roundtrip_and_batch():  # test_spectral.cpp:64-71
    for n in (8, 64, 512, 4096):
        x = rnd(3 * n, 200 + n).reshape(3, n).astype(np.float32)
        back = T.inverse_real(T.forward_real(x), n)
        assert np.abs(back - x).max() < 5e-6


def test_circular_conv_and_mac():  # test_spectral.cpp:96-141
    for n in (8, 16, 32):
        x, h = rnd(n, 300 + n), rnd(n, 400 + n)
        prod = T.mac(np.zeros(n // 2 + 1, complex), T.forward_real(x), T.forward_real(h))
        ref = O.inverse_real(O.mac(np.zeros(n // 2 + 1, complex), O.forward_real(x), O.forward_real(h)))
        assert np.abs(T.inverse_real(prod, n) - ref).max() < 1e-5
    g = np.random.default_rng(5)
    f = lambda: (g.uniform(-1, 1, 33) + 1j * g.uniform(-1, 1, 33)).astype(np.complex64)  # noqa: E731
    acc, a, b = f(), f(), f()
    assert np.abs(T.mac(acc, a, b) - (acc + a * b)).max() < 1e-6


def test_spectral_validation():  # test_spectral.cpp:143-161
    for n in (4, 12):
        with pytest.raises(T.InvalidSizeError):
            T.forward_real(np.zeros(n))
    bad = np.zeros(9, complex)
    bad[0] = 1e-3j
    with pytest.raises(T.InvalidSpectrumError):
        T.inverse_real(bad, 16)
    bad = np.zeros(9, complex)
    bad[8] = 1e-3j
    with pytest.raises(T.InvalidSpectrumError):
        T.inverse_real(bad, 16)
    with pytest.raises(T.InvalidSizeError):
        T.inverse_real(np.zeros(4, complex), 16)


def test_window():  # test_partition.cpp:25-47
    w = T.hann_window(256)
    assert w[0] == 0 and w[256] == 2.0
    assert np.abs(w.astype(np.float64) - O.hann_window(256)).max() < 1e-7
    with pytest.raises(T.InvalidSizeError):
        T.hann_window(1)


# ------------------------------------------------------------ partition
@pytest.mark.parametrize("hop,n_ir,minp", [(256, 2048, 1), (128, 700, 1), (256, 512, 4), (16, 1, 1), (512, 32768, 1)])
def test_partition_vs_oracle(hop, n_ir, minp):  # partition.cpp:20-51; test_partition.cpp:49-122
    ir = rnd(n_ir, n_ir + hop).astype(np.float32)
    g = T.partition(ir, hop, minp)
    o = O.partition(ir.astype(np.float64), hop, minp)
    assert g.partition_count == o.partition_count
    gs, os_ = g.spectra(), o.spectra()
    assert np.abs(gs - os_).max() < 3e-6 * np.sqrt(2 * hop)
    if minp > 1:
        assert np.abs(gs[0, 1:]).max() == 0.0


def test_partition_validation():  # test_partition.cpp:124-130
    with pytest.raises(T.InvalidInputError):
        T.partition(np.zeros((0, 1)), 256)
    for hop in (0, 24, 1):
        with pytest.raises(T.InvalidSizeError):
            T.partition(rnd(64, 15), hop)


# ------------------------------------------------------------ engine
def test_engine_geometry():  # test_engine.cpp:42-58
    one = T.TvolapEngine(T.partition(delta_ir(1, 1), 256))
    assert (one.partition_count(), one.latency(), one.switching_latency(), one.delay_line_depth()) == (1, 512, 256, 1)
    four = T.TvolapEngine(T.partition(delta_ir(1, 2048), 256))
    assert (four.partition_count(), four.delay_line_depth(), four.hop(), four.channels()) == (4, 7, 256, 1)
    big = T.TvolapEngine(T.partition(delta_ir(1, 32768), 512))
    assert big.partition_count() == 32 and big.switching_latency() == 512 and big.stream_delay() == 512


def test_zero_stays_zero_after_reset():  # test_engine.cpp:60-69
    eng = T.TvolapEngine(T.partition(delta_ir(1, 1024), 128))
    z = np.zeros((128, 1))
    for _ in range(5):
        assert np.abs(eng.process(z)).max() == 0.0
    eng.process(rnd(128, 1, 1))
    eng.reset()
    for _ in range(5):
        assert np.abs(eng.process(z)).max() == 0.0


def test_identity_passthrough():  # test_engine.cpp:71-77
    eng = T.TvolapEngine(T.partition(delta_ir(1, 1), 16))
    x = rnd(128, 2, 1)
    assert np.abs(stream_through(eng, x, 128) - x).max() < 1e-6


@pytest.mark.parametrize("n_ir", [256, 512, 1024])
def test_fixed_filter_matches_oracle_and_linear_conv(n_ir):  # test_engine.cpp:79-89
    h, x = rnd(n_ir, 10 + n_ir), rnd(4 * n_ir, 20 + n_ir)
    y = stream_through(T.TvolapEngine(T.partition(h, 128)), x, x.size + n_ir - 1)[:, 0]
    ref = np.convolve(x.astype(np.float32).astype(np.float64), h.astype(np.float32).astype(np.float64))
    assert np.abs(y - ref).max() <= 1e-4 * np.abs(ref).max()
    yo = O.stream_through(O.Engine(O.partition(h.astype(np.float32), 128)), x.astype(np.float32), y.size)[:, 0]
    assert np.abs(y - yo).max() <= 1e-4 * np.abs(yo).max()


def test_channels_independent():  # test_engine.cpp:91-102
    ir, x = rnd(256, 30, 2), rnd(1024, 31, 2)
    eng = T.TvolapEngine(T.partition(ir, 64))
    assert eng.channels() == 2
    y = stream_through(eng, x, 1024 + 255)
    for c in range(2):
        ref = np.convolve(x[:, c], ir[:, c])
        assert np.abs(y[:, c] - ref).max() <= 1e-4 * np.abs(ref).max()


def test_engine_linear():  # test_engine.cpp:104-116
    s = T.partition(rnd(512, 40), 64)
    x1, x2 = rnd(512, 41), rnd(512, 42)
    a, b = 0.8, -2.5
    y1 = stream_through(T.TvolapEngine(s), x1, 900)
    y2 = stream_through(T.TvolapEngine(s), x2, 900)
    ym = stream_through(T.TvolapEngine(s), a * x1 + b * x2, 900)
    assert np.abs(ym - (a * y1 + b * y2)).max() < 1e-4 * np.abs(ym).max()


def test_constant_op_counts_through_exchange():  # test_engine.cpp:118-139
    a, b = T.partition(rnd(1024, 50), 128), T.partition(rnd(1024, 51), 128)
    eng = T.TvolapEngine(a)
    m = eng.partition_count()
    for i in range(12):
        if i == 6:
            eng.exchange_filter(b)
        eng.process(np.ones((128, 1)))
        c = eng.op_counts()
        assert (c.forward_transforms, c.inverse_transforms, c.spectral_macs) == (i + 1, i + 1, (i + 1) * m)


def test_exchange_identical_is_bit_identical():  # test_engine.cpp:141-157
    s = T.partition(rnd(512, 60), 64)
    x = rnd(1024, 61)
    plain, exch = T.TvolapEngine(s), T.TvolapEngine(s)
    for i in range(16):
        chunk = x[i * 64:(i + 1) * 64, None]
        y1 = plain.process(chunk)
        if i == 7:
            exch.exchange_filter(s)
        assert np.array_equal(y1, exch.process(chunk))


def test_polarity_flip_half_cosine():  # test_engine.cpp:159-188 (analytic known answer)
    hop, calls, switch_call = 256, 24, 12
    eng = T.TvolapEngine(T.partition(delta_ir(1, 2048), hop))
    stream = []
    for i in range(calls):
        if i == switch_call:
            eng.exchange_filter(T.partition(delta_ir(-1, 2048), hop))
        stream.append(eng.process(np.ones((hop, 1))))
    out = np.concatenate(stream)[hop:, 0].astype(np.float64)
    boundary = (switch_call - 1) * hop
    w = O.hann_window(hop)
    assert np.abs(out[2 * hop:boundary] - 1.0).max() < 1e-5
    assert np.abs(out[boundary:boundary + hop] - (0.5 * w[hop:] - 0.5 * w[:hop])).max() < 1e-5
    assert np.abs(out[boundary + hop:] + 1.0).max() < 1e-5
    assert abs(out[boundary + hop - 1] + 1.0) > 1e-5


def test_shorter_ir_via_min_partitions():  # test_engine.cpp:190-201
    long_ir, short_ir = rnd(512, 70), rnd(100, 71)
    eng = T.TvolapEngine(T.partition(long_ir, 64))
    assert eng.partition_count() == 4
    eng.exchange_filter(T.partition(short_ir, 64, eng.partition_count()))
    x = rnd(2048, 72)
    y = stream_through(eng, x, x.size + 99)[:, 0]
    ref = np.convolve(x, short_ir)
    assert np.abs(y - ref).max() <= 1e-4 * np.abs(ref).max()


def test_framing_and_compatibility_enforced():  # test_engine.cpp:203-216
    eng = T.TvolapEngine(T.partition(delta_ir(1, 512), 128))
    with pytest.raises(T.InvalidSizeError):
        eng.process(np.zeros((127, 1)))
    with pytest.raises(T.InvalidInputError):
        eng.process(np.zeros((128, 2)))
    for bad in (T.partition(delta_ir(1, 512), 64), T.partition(delta_ir(1, 2048), 128),
                T.partition(np.zeros((512, 2)) + np.eye(512, 2), 128)):
        with pytest.raises(T.IncompatibleFilterError):
            eng.exchange_filter(bad)
    with pytest.raises(T.InvalidConfigurationError):
        T.TvolapEngine(None)


def test_reset_keeps_staged_filter():  # test_engine.cpp:218-232
    eng = T.TvolapEngine(T.partition(delta_ir(1, 256), 64))
    eng.process(rnd(64, 80, 1))
    eng.exchange_filter(T.partition(delta_ir(-1, 256), 64))
    eng.reset()
    for _ in range(8):
        last = eng.process(np.ones((64, 1)))
    assert abs(last[63, 0] + 1.0) < 1e-5


def test_processor_facade():  # test_reference.cpp:254-266 (facade == raw engine)
    ir, x = rnd(1000, 3), rnd(64 * 20, 4)
    proc = T.make_processor("tvolap", ir, 64)
    eng = T.TvolapEngine(T.partition(ir, 64))
    for i in range(20):
        c = x[i * 64:(i + 1) * 64, None]
        assert np.array_equal(proc.process(c), eng.process(c))
    with pytest.raises(T.InvalidConfigurationError):
        T.make_processor("nope", ir, 64)
    proc.set_filter(rnd(900, 5))  # shorter IR: padded to M partitions
    with pytest.raises(T.IncompatibleFilterError):
        proc.set_filter(rnd(4096, 6))


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_cluster_sizes_agree(P):
    """Every cluster size (CTAs per lane, DSMEM gather) produces the oracle's output."""
    L, n_ir, S = 64, 1000, 3
    ir = rnd(n_ir, 12, S)
    x = rnd(L * 40, 13, S)
    eng = T.TvolapEngine(T.partition(ir, L))
    eng.set_launch_config(P, 128)
    y = stream_through(eng, x, x.shape[0])
    ref = O.stream_through(O.Engine(O.partition(ir.astype(np.float32), L)), x.astype(np.float32), x.shape[0])
    assert np.abs(y - ref).max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("hop", [2, 4, 8, 32, 1024])
def test_extreme_hops(hop):
    """Smallest/largest hops (4L = 8 .. 4096) against the oracle."""
    ir, x = rnd(3 * hop + 1, hop), rnd(12 * hop, hop + 1)
    y = stream_through(T.TvolapEngine(T.partition(ir, hop)), x, x.size)[:, 0]
    ref = O.stream_through(O.Engine(O.partition(ir.astype(np.float32), hop)), x.astype(np.float32), x.size)[:, 0]
    assert np.abs(y - ref).max() <= 1e-4 * np.abs(ref).max()


def test_process_hops_equals_process():
    """Multi-hop call == the same hops one process() at a time (bit-exact)."""
    ir, x = rnd(3000, 21, 4), rnd(128 * 30, 22, 4)
    s = T.partition(ir, 128)
    a, b = T.TvolapEngine(s), T.TvolapEngine(s)
    one = np.concatenate([a.process(x[i * 128:(i + 1) * 128]) for i in range(30)])  # (T, C)
    many = b.process_hops(np.ascontiguousarray(x.T))  # (C, T)
    # multi-hop calls run the hop-blocked kernel: same per-hop sums in the same order
    assert np.array_equal(one.T, many)
    b.set_block_config(0, 1 << 30)  # force the one-hop-at-a-time kernel for multi-hop calls
    c = T.TvolapEngine(s)
    c.set_block_config(0, 1 << 30)
    assert np.array_equal(one.T, c.process_hops(np.ascontiguousarray(x.T)))
    assert b.hops_processed() == 30


# ------------------------------------------------------------ hop-blocked kernel == hop-by-hop kernel
def _relerr(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("jb", [2, 4, 8, 16])
@pytest.mark.parametrize("hop,n_ir,P", [(64, 64, 1), (64, 200, 2), (32, 64 * 3, 4), (128, 3000, 1), (256, 32768, 4)])
def test_block_kernel_matches_streaming(jb, hop, n_ir, P):
    """process_hops (hop-blocked kernel, partial blocks, odd start) == process() hop by hop."""
    S = 3
    ir = rnd(n_ir, n_ir + jb, S)
    n = 3 * jb + 3
    x = rnd(hop * (n + 1), 7 + jb, S)
    s = T.partition(ir, hop)
    a, b = T.TvolapEngine(s), T.TvolapEngine(s)
    a.set_launch_config(P, 0)
    b.set_launch_config(P, 0)
    try:
        a.set_block_config(jb, 2)
        b.set_block_config(jb, 1 << 30)  # same partition grouping, but always the one-hop kernel
    except T.InvalidConfigurationError:
        pytest.skip("block does not fit in shared memory")
    ref = np.concatenate([b.process(x[i * hop:(i + 1) * hop]) for i in range(n + 1)])  # (T, S)
    xs = np.ascontiguousarray(x.T)
    first = a.process(x[:hop])  # one streaming hop first: the block starts at an odd hop
    rest = a.process_hops(xs[:, hop:])
    got = np.concatenate([first.T, rest], axis=1)
    assert np.array_equal(got, ref.T)


def test_block_kernel_with_exchanges_between_calls():
    hop, S = 64, 2
    sets = [T.partition(rnd(900, 40 + k, S), hop, 15) for k in range(4)]
    x = rnd(hop * 64, 99, S)
    a, b = T.TvolapEngine(sets[0]), T.TvolapEngine(sets[0])
    a.set_block_config(8, 2)
    b.set_block_config(8, 1 << 30)
    outs_a, outs_b = [], []
    for k in range(4):
        if k:
            a.exchange_filter(sets[k])
            b.exchange_filter(sets[k])
        seg = x[k * 16 * hop:(k + 1) * 16 * hop]
        outs_a.append(a.process_hops(np.ascontiguousarray(seg.T)))
        outs_b.append(np.concatenate([b.process(seg[i * hop:(i + 1) * hop]) for i in range(16)]).T)
    assert np.array_equal(np.concatenate(outs_a, 1), np.concatenate(outs_b, 1))


@pytest.mark.parametrize("ears", [1, 2])
@pytest.mark.parametrize("jb", [4, 16])
def test_block_kernel_bank_schedule(ears, jb):
    """Per-hop bank switching inside blocks (non-shared filters) == streaming kernel, ears share X."""
    hop, S, n_bank, n = 32, 5, 7, 41
    bank = rnd(n_bank * ears * 500, 5).reshape(n_bank, ears, 500)
    sched = np.random.default_rng(8).integers(0, n_bank, (n, S)).astype(np.int32)
    sched[:10] = 3  # a run of shared filters
    x = np.ascontiguousarray(rnd(hop * n, 6, S).T)
    a = T.TvolapBankEngine(bank, hop, S)
    b = T.TvolapBankEngine(bank, hop, S)
    a.set_tuning("bank_pass", 0)  # the hop-blocked kernel itself (the bank pass: test_gpu_bank_pass.py)
    b.set_tuning("bank_pass", 0)
    a.set_block_config(jb, 2)
    b.set_block_config(jb, 1 << 30)  # never block, same partition grouping
    ya = a.process_hops(x, schedule=sched)
    yb = b.process_hops(x, schedule=sched)
    assert np.array_equal(ya, yb)
    # and against the oracle, ear by ear (error relative to the whole output's scale)
    scale = np.abs(ya).max()
    for s in range(S):
        cur = None
        eng = None
        for h in range(n):
            if sched[h, s] != cur:
                st = O.partition(bank[sched[h, s]].T.astype(np.float32), hop)
                if eng is None:
                    eng = O.Engine(st)
                else:
                    eng.exchange_filter(st)
                cur = sched[h, s]
            seg = np.repeat(x[s, h * hop:(h + 1) * hop, None].astype(np.float64), ears, axis=1)
            yo = eng.process(seg)
            for e in range(ears):
                assert np.abs(ya[s * ears + e, h * hop:(h + 1) * hop] - yo[:, e]).max() <= 1e-4 * scale


# ------------------------------------------------------------ frame adapter (test_adapter.cpp)
def test_adapter_arbitrary_chunking_is_bit_exact():  # test_adapter.cpp:38-63
    hop, total = 128, 2048
    ir, x = rnd(512, 1), rnd(total, 2, 1)
    strict = T.TvolapProcessor(ir, hop)
    ref = np.concatenate([strict.process(x[i * hop:(i + 1) * hop]) for i in range(total // hop)])
    chunked = T.TvolapProcessor(ir, hop)
    ad = T.FrameAdapter(chunked)
    g = np.random.default_rng(3)
    got, fed = [], 0
    while fed < total:
        n = min(int(g.integers(0, 700)), total - fed)
        got.append(ad.push(x[fed:fed + n]))
        fed += n
    out = np.concatenate(got)
    assert out.shape[0] == total and ad.buffered() == 0
    assert np.array_equal(out, ref)


def test_adapter_flush_zero_pads():  # test_adapter.cpp:65-90
    hop = 64
    proc = T.TvolapProcessor(delta_ir(1, 1), hop)
    ad = T.FrameAdapter(proc)
    x = rnd(100, 4, 1)
    first = ad.push(x)
    assert first.shape[0] == 64 and ad.buffered() == 36
    rest = ad.flush()
    assert rest.shape[0] == 64 and ad.buffered() == 0
    stream = np.concatenate([first, rest])[:, 0]
    assert np.abs(stream[:64]).max() < 1e-6
    assert np.abs(stream[64:100] - x[:36, 0]).max() < 1e-6  # identity, stream delay one hop
    assert ad.flush().shape[0] == 0
    with pytest.raises(T.InvalidInputError):
        ad.push(np.zeros((10, 2)))


@pytest.mark.parametrize("S", [3, 64])
def test_bank_engine_single_hop_select(S):
    """process() on a bank engine uses the latched select_bank choice (== per-hop schedule)."""
    hop, n_bank, n = 32, 6, 12
    bank = rnd(n_bank * 300, 17).reshape(n_bank, 1, 300)
    sched = np.random.default_rng(9).integers(0, n_bank, (n, S)).astype(np.int32)
    x = rnd(hop * n, 18, S)
    a, b = T.TvolapBankEngine(bank, hop, S), T.TvolapBankEngine(bank, hop, S)
    b.set_tuning("bank_pass", 0)  # the hop kernels: bit-identical to process() per hop
    ya = []
    for h in range(n):
        a.select_bank(sched[h])
        ya.append(a.process(x[h * hop:(h + 1) * hop]))
    ya = np.concatenate(ya).T
    yb = b.process_hops(np.ascontiguousarray(x.T), schedule=sched)
    assert np.array_equal(ya, yb)
    c = T.TvolapBankEngine(bank, hop, S)  # default: the bank pass, equal to fp32 rounding
    yc = c.process_hops(np.ascontiguousarray(x.T), schedule=sched)
    assert c.wide_passes() >= 1
    assert np.abs(yc - ya).max() <= 2e-6 * np.abs(ya).max()
    with pytest.raises(T.InvalidInputError):
        a.select_bank(np.full(S, n_bank, np.int32))


@pytest.mark.parametrize("hop,ears,S,n_bank", [(32, 1, 300, 7), (128, 2, 96, 5)])
def test_bank_engine_entry_order(hop, ears, S, n_bank):
    """The one-hop kernel visits the sources grouped by their bank entry (tuning entry_order=1,
    default): only the CTA order changes, so the outputs equal the source-order launch bit for bit,
    after select_bank and after a schedule call whose last row becomes the selection."""
    n = 10
    bank = rnd(n_bank * ears * 900, 27).reshape(n_bank, ears, 900)
    sched = np.random.default_rng(29).integers(0, n_bank, (2 * n, S)).astype(np.int32)
    x = rnd(hop * 2 * n, 28, S)
    ys = []
    for order in (1, 0):
        e = T.TvolapBankEngine(bank, hop, S)
        e.set_tuning("entry_order", order)
        y = []
        for h in range(n):
            e.select_bank(sched[h])
            y.append(e.process(x[h * hop:(h + 1) * hop]))
        y.append(e.process_hops(np.ascontiguousarray(x[n * hop:(2 * n - 1) * hop].T), schedule=sched[n:2 * n - 1]).T)
        y.append(e.process(x[(2 * n - 1) * hop:]))  # the schedule's last row is the latched selection
        ys.append(np.concatenate(y))
    assert np.array_equal(ys[0], ys[1])


@pytest.mark.parametrize("hop,ears,S,taps", [(32, 1, 300, 32 * 64), (128, 2, 96, 128 * 16), (32, 2, 40, 900)])
def test_one_hop_kernel_threads_per_cta(hop, ears, S, taps):
    """Threads per CTA of the one-hop kernel (tuning nt; automatic rule: one thread per (partition
    group, float4 column), two-warp CTAs for bank engines whose slice is one warp wide, like C5):
    fewer threads make each MAC thread walk several columns of its group, more leave threads idle
    in the MAC — the partition groups and the summation order do not change, so every geometry
    gives the same bits as the automatic one (engine.cpp:85-92 sums over m in one fixed order)."""
    n, n_bank = 12, 5
    bank = rnd(n_bank * ears * taps, 31).reshape(n_bank, ears, taps)
    sched = np.random.default_rng(33).integers(0, n_bank, (n, S)).astype(np.int32)
    x = rnd(hop * n, 32, S)
    ys = []
    for nt in (0, 32, 64, 128, 256, 512):
        e = T.TvolapBankEngine(bank, hop, S)
        e.set_tuning("bank_pass", 0)
        if nt:
            e.set_tuning("nt", nt)
        y = []
        for h in range(n):
            e.select_bank(sched[h])
            y.append(e.process(x[h * hop:(h + 1) * hop]))
        ys.append(np.concatenate(y))
    for y in ys[1:]:
        assert np.array_equal(ys[0], y)
    # the launch-config call reports what the one-hop launch uses, and an override is honoured
    e = T.TvolapBankEngine(bank, hop, S)
    auto = e.launch_config()[1]
    assert (auto <= 64) if hop == 32 else (auto == 256)
    e.set_launch_config(0, 128)
    assert e.launch_config()[1] == 128
    e.select_bank(sched[0])
    assert np.array_equal(e.process(x[:hop]), ys[0][:hop])


def test_cpp_wrapper():
    """The C++ drop-in (include/tvolap_b200.hpp) runs the reference's engine tests on the GPU:
    tests/cpp/test_wrapper.cpp, built by _build.build() into lib/test_wrapper; exit 0 = PASS."""
    import subprocess
    from pathlib import Path

    exe = Path(T.__file__).resolve().parent / "lib" / "test_wrapper"
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


def test_prebuilt_set_exchange_is_o1_and_shared():
    """exchange_filter(shared_ptr<const FilterPartitionSet>) (engine.hpp:55) launches no K4: the
    engine reads the set's device spectra in place; sets are shared between engines; reassemble
    (partition.cpp:53-65) gives the response back, zero-padded to M*2L taps."""
    hop = 64
    g = np.random.default_rng(12)
    sets = [T.partition(g.standard_normal((1500, 3)) * 0.1, hop) for _ in range(3)]
    a, b = T.TvolapEngine(sets[0]), T.TvolapEngine(sets[0])
    x = g.uniform(-1, 1, (hop * 20, 3))
    a.process(x[:hop])
    b.process(x[:hop])
    n0 = a.kernel_launches()
    a.exchange_filter(sets[1])
    a.exchange_filter(sets[2])  # last staged wins
    ya = a.process(x[hop:2 * hop])
    assert a.kernel_launches() - n0 == 1
    b.exchange_filter(sets[2])
    yb = b.process(x[hop:2 * hop])
    assert np.array_equal(ya, yb)
    back = T.reassemble(sets[1])
    assert back.shape == (2 * hop * sets[1].partition_count, 3)
    assert np.abs(back[:1500] - sets[1].taps.T).max() <= 1e-5 * np.abs(sets[1].taps).max()
    assert np.abs(back[1500:]).max() <= 1e-6
    # a set transformed from taps (exchange_ir, side-stream K4) gives the same outputs as the set
    c = T.TvolapEngine(sets[0])
    c.process(x[:hop])
    c.exchange_ir(sets[2].taps)
    assert np.array_equal(c.process(x[hop:2 * hop]), ya)


def test_mix_group_single_rank_equals_device_mix():
    """tvolap_mix_group_* with world = 1 (no handles): scatter + rank-ordered gather = tvolap_mix_device,
    bit for bit (same source order), with a strided output buffer."""
    import ctypes

    import torch

    from paper_2310_00319_b200 import shard

    g = np.random.default_rng(5)
    S, E, n = 7, 2, 3000
    out = torch.from_numpy(g.standard_normal((S * E, n + 16)).astype(np.float32)).cuda()
    ref = torch.empty((E, n), device="cuda")
    T._check(T.lib().tvolap_mix_device(0, S, E, n, ctypes.c_void_p(out.data_ptr()), n + 16,
                                       ctypes.c_void_p(ref.data_ptr()), n, None))
    grp = shard.MixGroup(0, E, 4096)
    got = torch.empty((E, n), device="cuda")
    grp.allreduce(out, S, n, got)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    big = torch.zeros((S * E, 5000), device="cuda")
    with pytest.raises(T.InvalidSizeError):
        grp.allreduce(big, S, 5000, torch.empty((E, 5000), device="cuda"))  # more samples than the group holds
    grp.close()


@pytest.mark.parametrize("hop,ears,taps,S,variant", [(32, 1, 4096, 256, 1), (128, 2, 4096, 160, 2),
                                                     (32, 2, 8192, 160, 3), (128, 1, 4096, 256, 1)])
def test_one_hop_ring_kernel_is_bit_identical(hop, ears, taps, S, variant):
    """Bank engines' process() on the persistent bulk-copy ring kernel (cp.async.bulk + mbarrier
    stages running ahead across sources; opt-in, tuning hop_ring = 1..4) against the default hop kernel:
    same partition groups and summation order, so every output bit agrees — over enough hops to
    wrap the delay line, with the selection changing every hop, and vs the reference."""
    import oracle as O
    from parity import TOL, best_oracle

    g = np.random.default_rng(hop + ears)
    n_bank = 6
    bank = (g.standard_normal((n_bank, ears, taps)) * np.exp(-np.arange(taps) / (taps / 5))).astype(np.float32)
    a = T.TvolapBankEngine(bank, hop, S)
    a.set_tuning("hop_ring", variant)  # one of the four ring geometries (opt-in: default 0)
    b = T.TvolapBankEngine(bank, hop, S)
    assert b.get_tuning("hop_ring") == 0
    M = a.partition_count()
    n = 2 * M + 21  # the 2M-1 deep delay line wraps
    x = g.uniform(-1, 1, (S, n * hop)).astype(np.float32)
    sel = g.integers(0, n_bank, (n, S)).astype(np.int32)
    ya, yb = [], []
    for h in range(n):
        blk = np.ascontiguousarray(x[:, h * hop:(h + 1) * hop].T)
        a.select_bank(sel[h])
        b.select_bank(sel[h])
        ya.append(a.process(blk).T)
        yb.append(b.process(blk).T)
    assert a.ring_launches() == n and b.ring_launches() == 0
    ya, yb = np.concatenate(ya, 1), np.concatenate(yb, 1)
    assert np.array_equal(ya, yb)
    with O.using(best_oracle()):
        _, ref = O.run_workload(hop, M, S, ears, n, x.astype(np.float64), 1, bank_ir=bank.astype(np.float64),
                                schedule=sel, threads=8)
    assert np.abs(ya - ref).max() <= TOL * np.abs(ref).max()
    # mixed with multi-hop calls (bank pass / hop-blocked kernel) the stream continues seamlessly
    c = T.TvolapBankEngine(bank, hop, S)
    c.set_tuning("hop_ring", 1)
    half = n // 2
    y1 = c.process_hops(x[:, : half * hop], schedule=sel[:half])
    tail = []
    for h in range(half, n):
        c.select_bank(sel[h])
        tail.append(c.process(np.ascontiguousarray(x[:, h * hop:(h + 1) * hop].T)).T)
    yc = np.concatenate([y1] + tail, 1)
    assert c.ring_launches() == n - half
    assert np.abs(yc - ref).max() <= TOL * np.abs(ref).max()
