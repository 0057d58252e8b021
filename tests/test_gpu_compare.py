"""GPU comparison convolvers through the C-ABI: the reference's own
test_reference.cpp cases at fp32 tolerances, and parity with the fp64 oracle on seeded
multi-channel inputs across filter switches, per hop and as multi-hop calls."""
import ctypes

import numpy as np
import pytest

import oracle as O
from paper_2310_00319_b200 import tvolap as T

pytestmark = pytest.mark.gpu
TOL = 1e-4  # north-star bound, relative to the reference output's scale


def rnd(rows, cols, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (rows, cols))


def delta(gain, n, delay=0, ch=1):
    h = np.zeros((n, ch))
    h[delay, :] = gain
    return h


def stream_through(proc, x, n_out):
    hop = proc.hop()
    calls = -(-(n_out + proc.stream_delay()) // hop)
    padded = np.zeros((calls * hop, x.shape[1]))
    padded[: x.shape[0]] = x
    out = np.concatenate([proc.process(padded[i * hop:(i + 1) * hop]) for i in range(calls)])
    return out[proc.stream_delay(): proc.stream_delay() + n_out]


def test_direct_form_prefix():  # test_reference.cpp:71-79
    ir, x = rnd(33, 1, 6), rnd(256, 1, 7)
    proc = T.DirectProcessor(ir, 64)
    assert proc.latency() == 0
    y = stream_through(proc, x, 256)
    assert np.abs(y[:, 0] - np.convolve(x[:, 0], ir[:, 0])[:256]).max() < 1e-5


def test_block_convolvers_match_brute_force():  # :81-95
    h, x = rnd(256, 1, 8)[:, 0], rnd(2000, 1, 9)
    ref = np.convolve(x[:, 0], h)
    for name in ("ola", "ols"):
        proc = T.make_processor(name, h, 0)
        assert proc.hop() == 256 and proc.latency() == 256
        y = stream_through(proc, x, ref.size)
        assert np.abs(y[:, 0] - ref).max() < 1e-4 * np.abs(ref).max()


def test_wola_identity_and_approximation():  # :97-120
    proc = T.WolaProcessor(delta(1.0, 256))
    assert (proc.hop(), proc.latency(), proc.stream_delay(), proc.switching_latency()) == (128, 256, 128, 128)
    x = rnd(1500, 1, 10)
    assert np.abs(stream_through(proc, x, 1500) - x).max() < 1e-5
    q = 10
    proc = T.WolaProcessor(delta(1.0, 256, q))
    x = rnd(1000, 1, 11)
    want = np.zeros((1000, 1))
    want[q:] = x[: 1000 - q]
    err = np.abs(stream_through(proc, x, 1000) - want).max()
    assert 1e-4 < err < 1e-1


@pytest.mark.parametrize("shape", [T.CrossfadeConfig.HANN, T.CrossfadeConfig.LINEAR])
def test_crossfade_curve(shape):  # :122-152
    hop, dur = 64, 128
    ones = np.ones((hop, 1))
    proc = T.CfTdcProcessor(delta(1.0, 8), hop, T.CrossfadeConfig(dur, shape))
    out = []
    for i in range(12):
        if i == 4:
            proc.switch_filter(delta(-1.0, 8), T.CrossfadeConfig(dur, shape))
        out.append(proc.process(ones))
    out = np.concatenate(out)[:, 0]
    b, t = 4 * hop, np.arange(dur)
    g = 0.5 * (1 - np.cos(np.pi * t / dur)) if shape == T.CrossfadeConfig.HANN else t / dur
    assert np.abs(out[:b] - 1.0).max() < 1e-6
    assert np.abs(out[b:b + dur] - (1.0 - 2.0 * g)).max() < 1e-6
    assert np.abs(out[b + dur:] + 1.0).max() < 1e-6


def test_crossfade_switch_rules():  # :154-196
    hop = 32
    x = rnd(hop * 10, 1, 12)
    proc = T.CfTdcProcessor(delta(1.0, 4), hop, T.CrossfadeConfig(97))
    out = []
    for i in range(10):
        if i == 2:
            proc.set_filter(delta(1.0, 4))
        out.append(proc.process(x[i * hop:(i + 1) * hop]))
    assert np.abs(np.concatenate(out) - x).max() < 1e-6  # complementary gains
    proc = T.CfTdcProcessor(delta(1.0, 8), hop, T.CrossfadeConfig(200, T.CrossfadeConfig.LINEAR))
    ones = np.ones((hop, 1))
    proc.process(ones)
    proc.set_filter(delta(0.5, 8))
    with pytest.raises(T.SwitchInProgressError):
        proc.set_filter(delta(0.25, 8))
    proc.process(ones)
    assert proc.fading()
    for _ in range(8):
        proc.process(ones)
    assert not proc.fading()
    proc.set_filter(delta(0.25, 8))
    hard = T.CfTdcProcessor(delta(1.0, 4), 16, T.CrossfadeConfig(1))
    o = []
    for i in range(6):
        if i == 3:
            hard.set_filter(delta(-1.0, 4))
        o.append(hard.process(np.ones((16, 1))))
    o = np.concatenate(o)[:, 0]
    assert o[47] == pytest.approx(1.0) and o[48] == pytest.approx(-1.0)


@pytest.mark.parametrize("name", ["ola", "ols"])
def test_block_switch_transition(name):  # :198-233
    n = 256
    old_ir, new_ir = delta(0.5, n, 100), delta(1.0, n)
    x = rnd(8 * n, 1, 13)
    sw, fr = T.make_processor(name, old_ir, 0), T.make_processor(name, new_ir, 0)
    out_s, out_f = [], []
    for i in range(8):
        if i == 4:
            sw.set_filter(new_ir)
        out_s.append(sw.process(x[i * n:(i + 1) * n]))
        out_f.append(fr.process(x[i * n:(i + 1) * n]))
    diff = np.abs(np.concatenate(out_s) - np.concatenate(out_f))[:, 0]
    if name == "ola":
        assert diff[4 * n:5 * n].max() > 1e-3
        assert diff[-3 * n:].max() < 1e-6
    else:
        assert diff[-4 * n:].max() < 1e-6


def test_factory_and_validation():  # :235-252
    ir = delta(1.0, 512)
    assert T.make_processor("tdc", ir, 128).name() == "tdc"
    assert T.make_processor("cf-tdc", ir, 128).switching_latency() == 128
    assert T.make_processor("ola", ir, 0).hop() == 512
    assert T.make_processor("ols", ir, 0).latency() == 512
    assert T.make_processor("wola", ir, 0).hop() == 256
    tv = T.make_processor("tvolap", ir, 128)
    assert tv.latency() == 256 and tv.stream_delay() == 128
    with pytest.raises(T.InvalidConfigurationError):
        T.make_processor("nope", ir, 128)
    proc = T.make_processor("ola", delta(1.0, 64), 0)
    with pytest.raises(T.InvalidSizeError):
        proc.process(np.zeros((63, 1)))
    with pytest.raises(T.InvalidInputError):
        proc.process(np.zeros((64, 2)))
    with pytest.raises(T.InvalidSizeError):
        T.OlaProcessor(delta(1.0, 100))
    with pytest.raises(T.IncompatibleFilterError):
        proc.set_filter(delta(1.0, 128))


def _oracle_proc(name, ir, hop, fade=None):
    if name == "cf-tdc":
        return O.Processor(name, ir, hop, fade.duration, fade.shape)
    return O.Processor(name, ir, hop)


def _gpu_proc(name, ir, hop, fade=None):
    return {"tdc": lambda: T.DirectProcessor(ir, hop), "cf-tdc": lambda: T.CfTdcProcessor(ir, hop, fade),
            "ola": lambda: T.OlaProcessor(ir), "ols": lambda: T.OlsProcessor(ir),
            "wola": lambda: T.WolaProcessor(ir)}[name]()


@pytest.mark.parametrize("name,taps,hop", [("tdc", 300, 64), ("cf-tdc", 300, 64), ("ola", 128, 0), ("ols", 256, 0),
                                           ("wola", 512, 0), ("ola", 2048, 0), ("tdc", 4096, 128)])
def test_parity_with_oracle_across_switches(name, taps, hop):
    """Seeded 3-channel input, a new filter every 5 hops, per-hop process() on the oracle vs
    multi-hop process_hops() calls on the GPU (calls break at the switches)."""
    ch, n_calls = 3, 5
    fade = T.CrossfadeConfig(hop + 17, T.CrossfadeConfig.HANN)
    irs = [rnd(taps, ch, 100 + k) * np.exp(-np.arange(taps) / (taps / 4))[:, None] for k in range(n_calls)]
    g = _gpu_proc(name, irs[0], hop, fade)
    o = _oracle_proc(name, irs[0], hop, fade)
    H = g.hop()
    x = rnd(H * 5 * n_calls, ch, 7)
    yg, yo = [], []
    for k in range(n_calls):
        if k:
            g.set_filter(irs[k])
            o.set_filter(irs[k])
        seg = x[k * 5 * H:(k + 1) * 5 * H]
        yg.append(g.process_hops(seg.T).T)
        yo.append(np.concatenate([o.process(seg[i * H:(i + 1) * H]) for i in range(5)]))
    yg, yo = np.concatenate(yg), np.concatenate(yo)
    assert np.abs(yg - yo).max() <= TOL * np.abs(yo).max(), name


@pytest.mark.parametrize("name", ["tdc", "cf-tdc", "ola", "ols", "wola"])
def test_multi_hop_equals_per_hop_and_reset(name):
    taps = 64 if name in ("tdc", "cf-tdc") else 128
    ir = rnd(taps, 2, 3)
    a = _gpu_proc(name, ir, 32, T.CrossfadeConfig(40))
    b = _gpu_proc(name, ir, 32, T.CrossfadeConfig(40))
    H = a.hop()
    x = rnd(H * 9, 2, 4)
    a.process_hops(rnd(H * 3, 2, 5).T)  # some history, then reset
    a.reset()
    ya = a.process_hops(x.T).T
    yb = np.concatenate([b.process(x[i * H:(i + 1) * H]) for i in range(9)])
    assert np.abs(ya - yb).max() <= 1e-6 * max(np.abs(yb).max(), 1.0)


def test_device_buffers():
    import torch

    ir = rnd(256, 2, 1)
    a, b = T.OlsProcessor(ir), T.OlsProcessor(ir)
    x = np.ascontiguousarray(rnd(256 * 4, 2, 2).T.astype(np.float32))
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    T._check(T.lib().tvolap_cmp_process_hops(a._h, ctypes.c_void_p(xd.data_ptr()), x.shape[1],
                                             ctypes.c_void_p(yd.data_ptr()), x.shape[1], 4))
    assert np.array_equal(yd.cpu().numpy(), b.process_hops(x))
