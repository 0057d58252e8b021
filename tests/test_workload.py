"""Host workload generators: determinism, distributions, and the bytes model."""
import numpy as np

from paper_2310_00319_b200 import workload as W


def test_white_is_deterministic_and_uniform():
    cfg = W.CONFIGS["C2"]
    a = W.white(cfg, 0, 4, 0, 20000)
    b = W.white(cfg, 0, 4, 0, 20000, threads=1)
    assert np.array_equal(a, b)
    assert a.min() >= -1 and a.max() < 1 and abs(a.mean()) < 0.02 and abs(a.var() - 1 / 3) < 0.01
    # windows of the same stream agree; lanes differ
    assert np.array_equal(W.white(cfg, 2, 1, 100, 50)[0], a[2, 100:150])
    assert not np.array_equal(a[0], a[1])
    d = W.white(cfg, 0, 1, 0, 100, dtype=np.float64)
    assert np.array_equal(d[0], a[0, :100].astype(np.float64))


def test_uniform_mapping_matches_reference_formula():
    """signal_gen.cpp:14-16: 2 * ((g() >> 11) * 2^-53) - 1 on the 64-bit word."""
    cfg = W.CONFIGS["C1"]
    r = W.wlib().tv_rand64_c(cfg.seed, (1 << 60) | 0, 5)
    v = 2.0 * ((r >> 11) * 2.0 ** -53) - 1.0
    assert np.float32(v) == W.white(cfg, 0, 1, 5, 1)[0, 0]


def test_irs_unit_energy_decay_and_t60_range():
    cfg = W.CONFIGS["C2"]
    irs = W.fresh_irs(cfg, 3, 0, 4, dtype=np.float64)
    assert irs.shape == (4, 1, 32768)
    e = (irs ** 2).sum(-1)
    assert np.allclose(e, 1.0, rtol=1e-6)
    for l in range(4):
        t = W.t60_of(cfg, l, 3)
        assert 0.3 <= t <= 1.5
    # decaying envelope: energy of the first quarter dominates the last quarter
    assert ((irs[..., :8192] ** 2).sum() > 10 * (irs[..., -8192:] ** 2).sum())
    assert np.array_equal(W.fresh_irs(cfg, 3, 1, 1), W.fresh_irs(cfg, 3, 0, 4)[1:2])


def test_schedules():
    c1 = W.CONFIGS["C1"]
    s = W.schedule(c1, 0, 200)
    assert s.shape == (200, 1) and set(np.unique(s)) == {0, 1}
    assert (s[:64] == 0).all() and (s[64:128] == 1).all()
    c5 = W.CONFIGS["C5"]
    s5 = W.schedule(c5, 10, 50)
    assert s5.shape == (50, 4096) and s5.min() >= 0 and s5.max() < 1024
    assert np.array_equal(W.schedule(c5, 10, 50, lane0=100, lanes=5), s5[:, 100:105])
    assert np.array_equal(W.schedule(c5, 12, 2), s5[2:4])


def test_bytes_model_matches_baseline_table():
    """SURVEY.md §8(d) compulsory MB/hop column (C2 34.8, C4 1084.2)."""
    assert abs(W.bytes_per_hop(W.CONFIGS["C2"]) / 1e6 - 34.8) < 0.1
    assert abs(W.bytes_per_hop(W.CONFIGS["C4"]) / 1e6 - 1084.2) < 0.5
    assert W.CONFIGS["C2"].hops == 5625 and W.CONFIGS["C5"].hops == 15000
