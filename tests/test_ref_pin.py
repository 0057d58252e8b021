"""Pin the restated oracle to the REFERENCE ITSELF.

oracle/_ref/libtvolap_ref.so is the reference's own proj/src/{spectral,partition,engine}.cpp,
compiled unmodified from /root/reference against the minimal Eigen stand-in
(oracle/eigen_shim, recipe oracle/Makefile `ref`, harness oracle/ref_harness.cpp). Every case
below runs the same call on the port (oracle/tvolap_oracle.cpp) and on the reference and asserts
the outputs are BIT-IDENTICAL: same table formulas, same DIT order, same untangle, same ring
indexing, same hop-2 overlap-add, same error classes. The GPU parity tests then check the CUDA
path against this pinned oracle (and against _ref directly where it is present, tests/parity.py).
"""
import numpy as np
import pytest

import oracle as O
from paper_2310_00319_b200 import workload as W
from parity import oracle_config

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def both(fn):
    with O.using("port"):
        a = fn()
    with O.using("ref"):
        b = fn()
    return a, b


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    assert np.array_equal(a, b), f"max |diff| {np.abs(a - b).max()}"


@pytest.mark.parametrize("n", [8, 16, 64, 128, 256, 512, 1024, 2048, 4096])
def test_forward_inverse_bit_exact(n):
    g = np.random.default_rng(n)
    x = g.uniform(-1, 1, n)
    a, b = both(lambda: O.forward_real(x))
    same(a, b)
    spec = a.copy()
    a, b = both(lambda: O.inverse_real(spec, n))
    same(a, b)


def test_mac_and_window_bit_exact():
    g = np.random.default_rng(7)
    v = [g.normal(size=65) + 1j * g.normal(size=65) for _ in range(3)]
    for s in (v[0], v[1], v[2]):
        s[0] = s[0].real
        s[-1] = s[-1].real
    same(*both(lambda: O.mac(v[0], v[1], v[2])))
    for hop in (2, 32, 128, 256, 512):
        same(*both(lambda: O.hann_window(hop)))


@pytest.mark.parametrize("hop,taps,ch,minp", [(32, 32768, 2, 1), (128, 8192, 1, 1), (256, 1000, 3, 4), (2, 5, 1, 1)])
def test_partition_and_reassemble_bit_exact(hop, taps, ch, minp):
    ir = np.random.default_rng(hop + taps).normal(size=(taps, ch))

    def run():
        s = O.partition(ir, hop, minp)
        return (s.partition_count, s.channels, s.source_length, s.normalization_gain), s.spectra(), s.reassemble()

    (ga, sa, ra), (gb, sb, rb) = both(run)
    assert ga == gb
    same(sa, sb)
    same(ra, rb)


@pytest.mark.parametrize("case", [
    lambda: O.forward_real(np.ones(6)),          # InvalidSizeError
    lambda: O.inverse_real(np.array([1j, 2, 3, 4, 5]), 8),  # InvalidSpectrumError (DC imag)
    lambda: O.inverse_real(np.ones(4, complex), 8),         # InvalidSizeError (bin count)
    lambda: O.mac(np.ones(5), np.ones(9), np.ones(5)),      # InvalidSizeError
    lambda: O.hann_window(1),                                # InvalidSizeError
    lambda: O.partition(np.zeros((0, 1)), 4),                # InvalidInputError
    lambda: O.partition(np.ones(8), 3),                      # InvalidSizeError
    lambda: O.Engine(None),                                  # InvalidConfigurationError
])
def test_error_classes_match(case):
    codes = []
    for which in ("port", "ref"):
        with O.using(which):
            with pytest.raises(O.OracleError) as e:
                case()
            codes.append(e.value.code)
    assert codes[0] == codes[1]


def test_engine_errors_and_geometry_match():
    def run():
        out = []
        e = O.Engine(O.partition(np.ones((100, 2)), 8))
        out.append(tuple(e._geo()))
        for bad in (np.zeros((7, 2)), np.zeros((8, 3))):
            with pytest.raises(O.OracleError) as x:
                e.process(bad)
            out.append(x.value.code)
        for bad in (O.partition(np.ones((100, 2)), 4), O.partition(np.ones((400, 2)), 8),
                    O.partition(np.ones((100, 1)), 8)):
            with pytest.raises(O.OracleError) as x:
                e.exchange_filter(bad)
            out.append(x.value.code)
        return out

    a, b = both(run)
    assert a == b


def test_engine_stream_with_exchanges_reset_and_counts():
    """The engine API sequence of proj/tests/test_engine.cpp (exchange between hops, last staged
    wins, staged survives reset) on both libraries, hop by hop, bit for bit."""
    g = np.random.default_rng(3)
    hop, taps, ch = 16, 300, 3
    irs = [g.normal(size=(taps, ch)) for _ in range(4)]
    x = g.uniform(-1, 1, (hop * 60, ch))

    def run():
        e = O.Engine(O.partition(irs[0], hop))
        outs = []
        for k in range(60):
            if k == 10:
                e.exchange_filter(O.partition(irs[1], hop))
            if k == 25:
                e.exchange_filter(O.partition(irs[2], hop))
                e.exchange_filter(O.partition(irs[3], hop))  # last staged wins
            if k == 40:
                e.exchange_filter(O.partition(irs[1], hop))
                e.reset()  # staged filter survives reset
            outs.append(e.process(x[k * hop:(k + 1) * hop]))
        return np.concatenate(outs), e.op_counts()

    (ya, ca), (yb, cb) = both(run)
    same(ya, yb)
    assert ca == cb


# Every BASELINE config's own geometry, workload generators and switch schedule, on a prefix of
# >= 2(2M-1) hops for the small-M configs (the ring wraps) and across several switches for all.
@pytest.mark.parametrize("name,hops,sources", [
    ("C1", 400, None),   # 2 IRs alternating every 64 hops, ring (63 slots) wrapped 6x
    ("C2", 260, 2),      # fresh IR every 16 hops, 16 switches, ring (127 slots) wrapped
    ("C3", 520, 3),      # per-hop bank choice, 2 ears, ring (255 slots) wrapped
    ("C4", 1030, 1),     # fresh IR every 8 hops, 128 switches, L=512 M=256, ring (511 slots) wrapped
    ("C5", 1100, 2),     # per-hop bank choice from 1024, ring (1023 slots) wrapped
])
def test_config_workloads_bit_exact(name, hops, sources):
    cfg = W.CONFIGS[name]
    ya = oracle_config(cfg, hops, sources=sources, which="port")
    yb = oracle_config(cfg, hops, sources=sources, which="ref")
    same(ya, yb)
    assert np.abs(ya).max() > 0
