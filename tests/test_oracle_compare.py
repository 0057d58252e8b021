"""Pins the oracle's comparison convolvers to the reference's own tests:
proj/tests/test_reference.cpp:71-252, same inputs' shapes, same tolerances."""
import numpy as np
import pytest

from oracle import HANN, LINEAR, OracleError, Processor, make_processor


def rnd(rows, cols, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (rows, cols))


def delta(gain, n, delay=0):
    h = np.zeros((n, 1))
    h[delay, 0] = gain
    return h


def stream_through(proc, x, n_out):  # test_reference.cpp:25-35
    hop = proc.hop()
    total = n_out + proc.stream_delay()
    calls = -(-total // hop)
    padded = np.zeros((calls * hop, x.shape[1]))
    padded[: x.shape[0]] = x
    out = np.concatenate([proc.process(padded[i * hop:(i + 1) * hop]) for i in range(calls)])
    return out[proc.stream_delay(): proc.stream_delay() + n_out]


def test_streaming_direct_form_reproduces_the_convolution_prefix():  # :71-79
    ir = rnd(33, 1, 6)
    x = rnd(256, 1, 7)
    proc = Processor("tdc", ir, 64)
    assert proc.latency() == 0
    y = stream_through(proc, x, 256)
    assert np.abs(y[:, 0] - np.convolve(x[:, 0], ir[:, 0])[:256]).max() < 1e-12


def test_block_convolvers_match_brute_force():  # :81-95
    h = rnd(256, 1, 8)[:, 0]
    x = rnd(2000, 1, 9)
    ref = np.convolve(x[:, 0], h)
    for name in ("ola", "ols"):
        proc = make_processor(name, h, 0)
        assert proc.hop() == 256 and proc.latency() == 256
        y = stream_through(proc, x, ref.size)
        assert np.abs(y[:, 0] - ref).max() < 1e-9


def test_wola_reconstructs_through_identity():  # :97-106
    proc = Processor("wola", delta(1.0, 256))
    assert (proc.hop(), proc.latency(), proc.stream_delay(), proc.switching_latency()) == (128, 256, 128, 128)
    x = rnd(1500, 1, 10)
    assert np.abs(stream_through(proc, x, 1500) - x).max() < 1e-9


def test_wola_is_only_approximate_for_a_general_filter():  # :108-120
    q = 10
    proc = Processor("wola", delta(1.0, 256, q))
    x = rnd(1000, 1, 11)
    y = stream_through(proc, x, 1000)
    want = np.zeros((1000, 1))
    want[q:] = x[: 1000 - q]
    err = np.abs(y - want).max()
    assert 1e-4 < err < 1e-1


@pytest.mark.parametrize("shape", [HANN, LINEAR])
def test_crossfade_follows_the_gain_curve(shape):  # :122-152
    hop, dur = 64, 128
    ones = np.ones((hop, 1))
    proc = Processor("cf-tdc", delta(1.0, 8), hop, dur, shape)
    out = []
    for i in range(12):
        if i == 4:
            proc.switch_filter(delta(-1.0, 8), dur, shape)
        out.append(proc.process(ones))
    out = np.concatenate(out)[:, 0]
    b = 4 * hop
    assert np.allclose(out[:b], 1.0, rtol=1e-12)
    t = np.arange(dur)
    g = 0.5 * (1 - np.cos(np.pi * t / dur)) if shape == HANN else t / dur
    assert np.allclose(out[b:b + dur], 1.0 - 2.0 * g, rtol=1e-12, atol=1e-14)
    assert np.allclose(out[b + dur:], -1.0, rtol=1e-12)


def test_crossfade_gains_complementary():  # :154-166
    hop = 32
    x = rnd(hop * 10, 1, 12)
    proc = Processor("cf-tdc", delta(1.0, 4), hop, 97, HANN)
    out = []
    for i in range(10):
        if i == 2:
            proc.set_filter(delta(1.0, 4))
        out.append(proc.process(x[i * hop:(i + 1) * hop]))
    assert np.abs(np.concatenate(out) - x).max() < 1e-15


def test_crossfade_in_flight_rejects_another_switch():  # :168-182
    hop = 32
    proc = Processor("cf-tdc", delta(1.0, 8), hop, 200, LINEAR)
    ones = np.ones((hop, 1))
    proc.process(ones)
    proc.set_filter(delta(0.5, 8))
    with pytest.raises(OracleError) as e:
        proc.set_filter(delta(0.25, 8))
    assert e.value.code == 7
    proc.process(ones)
    assert proc.fading()
    with pytest.raises(OracleError):
        proc.set_filter(delta(0.25, 8))
    for _ in range(8):
        proc.process(ones)
    assert not proc.fading()
    proc.set_filter(delta(0.25, 8))


def test_duration_one_is_a_hard_switch():  # :184-196
    hop = 16
    proc = Processor("cf-tdc", delta(1.0, 4), hop, 1, HANN)
    ones = np.ones((hop, 1))
    out = []
    for i in range(6):
        if i == 3:
            proc.set_filter(delta(-1.0, 4))
        out.append(proc.process(ones))
    out = np.concatenate(out)[:, 0]
    assert out[3 * hop - 1] == pytest.approx(1.0) and out[3 * hop] == pytest.approx(-1.0)


@pytest.mark.parametrize("name", ["ola", "ols"])
def test_block_switch_transition(name):  # :198-233
    n = 256
    old_ir, new_ir = delta(0.5, n, 100), delta(1.0, n)
    x = rnd(8 * n, 1, 13 if name == "ola" else 14)
    sw, fr = Processor(name, old_ir), Processor(name, new_ir)
    out_s, out_f = [], []
    for i in range(8):
        if i == 4:
            sw.set_filter(new_ir)
        out_s.append(sw.process(x[i * n:(i + 1) * n]))
        out_f.append(fr.process(x[i * n:(i + 1) * n]))
    diff = np.abs(np.concatenate(out_s) - np.concatenate(out_f))[:, 0]
    b = 4 * n
    if name == "ola":
        assert diff[b:b + n].max() > 1e-3  # the outgoing filter's remainder is still audible
        assert diff[-3 * n:].max() < 1e-10
    else:
        assert diff[-4 * n:].max() < 1e-10


def test_factory_and_shape_validation():  # :235-252
    ir = delta(1.0, 512)
    assert make_processor("cf-tdc", ir, 128).switching_latency() == 128
    assert make_processor("ola", ir, 0).hop() == 512
    assert make_processor("ols", ir, 0).latency() == 512
    assert make_processor("wola", ir, 0).hop() == 256
    tv = make_processor("tvolap", ir, 128)
    assert tv.latency() == 256 and tv.stream_delay() == 128
    with pytest.raises(OracleError):
        make_processor("nope", ir, 128)
    proc = make_processor("ola", delta(1.0, 64), 0)
    with pytest.raises(OracleError) as e:
        proc.process(np.zeros((63, 1)))
    assert e.value.code == 1
    with pytest.raises(OracleError) as e:
        proc.process(np.zeros((64, 2)))
    assert e.value.code == 2
    with pytest.raises(OracleError) as e:
        Processor("ola", delta(1.0, 100))
    assert e.value.code == 1
