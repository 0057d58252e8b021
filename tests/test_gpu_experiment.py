"""Switch experiment on GPU output (proj/tests/test_experiment.cpp, acceptance.cpp crit 3/7)."""
import json

import numpy as np
import pytest

from paper_2310_00319_b200 import experiment as X
from paper_2310_00319_b200 import tvolap as T

pytestmark = pytest.mark.gpu


def delta(gain, n):
    h = np.zeros(n)
    h[0] = gain
    return h


def flip(hop, requested, n=8192):
    return X.run_switch(np.ones(n), delta(1, 2048), delta(-1, 2048), hop, requested)


def test_switch_quantizes_to_hop_boundaries():  # test_experiment.cpp:21-26
    assert flip(256, 300).metrics.switch_boundary == 256
    assert flip(256, 400).metrics.switch_boundary == 512
    assert flip(256, 0).metrics.switch_boundary == 0
    assert flip(256, 8191).metrics.switch_boundary == 7936


def test_polarity_flip_metrics():  # test_experiment.cpp:28-51
    run = flip(256, 3 * 256)
    m = run.metrics
    assert (m.algorithm, m.hop, m.audio_latency, m.stream_delay, m.switching_latency) == ("tvolap", 256, 512, 256, 256)
    assert m.switch_boundary == 768
    assert m.transition_start == 769
    assert m.transition_width == 256
    assert abs(m.max_step_transition - np.pi / 256) <= 0.01 * np.pi / 256
    assert m.max_step_steady < 1e-5
    u = np.arange(256)
    assert np.abs(run.output[768 + u, 0] - np.cos(np.pi * u / 256)).max() < 1e-5
    assert np.abs(run.old_ref[:, 0] - 1).max() < 1e-5 and np.abs(run.new_ref[:, 0] + 1).max() < 1e-5


def test_switch_width_and_validation():  # test_experiment.cpp:53-60,87-103
    assert flip(256, 4096).metrics.transition_width == 256
    ones = np.ones(4096)
    a, b = delta(1, 512), delta(-1, 512)
    with pytest.raises(T.InvalidInputError):
        X.run_switch(np.zeros((0, 1)), a, b, 128, 100)
    for bad in (4096, -1):
        with pytest.raises(T.InvalidConfigurationError):
            X.run_switch(ones, a, b, 128, bad)
    with pytest.raises(T.InvalidConfigurationError):
        X.run_switch(ones, a, b, 128, 100, input_rate=44100.0)
    assert X.run_switch(ones, a, delta(-1, 256), 128, 1024).metrics.transition_width == 128
    with pytest.raises(T.IncompatibleFilterError):
        X.run_switch(ones, a, delta(1, 4096), 128, 100)


def test_no_click_long_reverb_switch():  # acceptance.cpp:212-231 (crit 7), two-channel IRs
    g = np.random.default_rng(1)
    n_ir, hop = 32768, 512
    env = np.exp(-6.91 * np.arange(n_ir) / (0.3 * 44100))
    front = g.standard_normal((n_ir, 2)) * env[:, None]
    side = g.standard_normal((n_ir, 2)) * env[:, None]
    x = np.cumsum(g.standard_normal(65536)) * 1e-3  # band-limited (brown) input
    run = X.run_switch(x, front, side, hop, 32 * 1024, input_rate=44100.0, ir_a_rate=44100.0, ir_b_rate=44100.0)
    m = run.metrics
    assert m.switching_latency == 512 and m.switch_boundary == 32768
    steady = max(m.max_step_steady, np.abs(np.diff(run.old_ref, axis=0)).max(), np.abs(np.diff(run.new_ref, axis=0)).max())
    assert m.max_step_transition <= steady


def test_metric_tables_render():  # test_experiment.cpp:105-122
    run = flip(256, 768)
    rows = [run.metrics, flip(256, 2048).metrics]
    csv = X.metrics_csv(rows)
    assert csv == X.metrics_csv(rows)
    assert csv.startswith("algorithm,hop,audio_latency,stream_delay,switching_latency,switch_boundary,"
                          "transition_start,transition_width,max_step_transition,max_step_steady\n")
    assert "tvolap,256,512,256,256,768,769,256," in csv
    parsed = json.loads(X.metrics_json(rows))
    assert parsed[0]["transition_width"] == 256 and parsed[1]["switch_boundary"] == 2048
    tc = X.transition_csv(run, 4, 4).splitlines()
    assert tc[0] == "offset,output_0,old_ref_0,new_ref_0" and tc[1].startswith("-4,") and len(tc) == 9


def flip_alg(alg, hop, requested, n=8192, fade=None):
    return X.run_switch(np.ones(n), delta(1, 2048), delta(-1, 2048), hop, requested, alg, fade=fade)


def test_switch_widths_of_all_algorithms():  # test_experiment.cpp:53-60
    assert flip_alg("ols", 2048, 4096).metrics.transition_width == 0
    assert flip_alg("ola", 2048, 4096).metrics.transition_width == 0
    assert flip_alg("wola", 1024, 4096).metrics.transition_width == 1024
    assert flip_alg("tvolap", 256, 4096).metrics.transition_width == 256
    assert flip_alg("tdc", 256, 4096).metrics.transition_width == 0


def test_wola_crosses_over_along_half_cosine():  # test_experiment.cpp:62-71
    run = flip_alg("wola", 1024, 4096)
    b, r = run.metrics.switch_boundary, 1024
    u = np.arange(0, r, 7)
    assert np.abs(run.output[b + u, 0] - np.cos(np.pi * u / r)).max() < 1e-5


def test_crossfaded_direct_follows_requested_fade():  # test_experiment.cpp:73-85
    fade = T.CrossfadeConfig(512, T.CrossfadeConfig.LINEAR)
    run = X.run_switch(np.ones(8192), delta(1, 2048), delta(-1, 2048), 256, 2048, "cf-tdc", fade=fade)
    m = run.metrics
    assert (m.switching_latency, m.switch_boundary, m.transition_width) == (512, 2048, 512)
    u = np.arange(0, 512, 13)
    assert np.abs(run.output[2048 + u, 0] - (1.0 - 2.0 * u / 512)).max() < 1e-5


def test_engine_against_crossfaded_reference():  # test_experiment.cpp:136-171
    cmp = X.run_compare(np.ones(8192), delta(1, 2048), delta(-1, 2048), 256, 2048)
    assert cmp.metrics.fade_shape == "hann" and cmp.metrics.fade_duration == 256
    assert cmp.metrics.max_abs_diff < 1e-5  # the polarity flip: both transitions coincide
    # a smooth two-channel scene (stand-in for the reference's pink-noise binaural scene)
    g = np.random.default_rng(3)
    x = np.convolve(g.standard_normal(16384 + 63), np.hanning(64) / 32, mode="valid")
    t = np.arange(2048)[:, None]
    ir_a = g.standard_normal((2048, 2)) * np.exp(-t / 150.0)
    ir_b = g.standard_normal((2048, 2)) * np.exp(-t / 150.0)
    hann = X.run_compare(x, ir_a, ir_b, 256, 336)
    lin = X.run_compare(x, ir_a, ir_b, 256, 336, T.CrossfadeConfig.LINEAR)
    assert (hann.metrics.window_begin, hann.metrics.window_end) == (256, 256 + 3 * 256)
    assert hann.metrics.max_abs_diff > 0 and hann.metrics.output_rms > 0
    assert hann.metrics.diff_db < 0
    assert lin.metrics.fade_shape == "linear"
    csv = X.compare_csv([hann.metrics, lin.metrics])
    assert csv.startswith("fade_shape,fade_duration,window_begin,window_end,max_abs_diff,rms_diff,output_rms,diff_db\n")
    parsed = json.loads(X.compare_json([hann.metrics, lin.metrics]))
    assert parsed[0]["fade_shape"] == "hann" and parsed[1]["fade_shape"] == "linear"
