"""WAV I/O (proj/tests/test_wav.cpp) on CPU, and the CLI `process` path on the GPU
(proj/tests/CMakeLists.txt CLI round-trips)."""
import struct
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2310_00319_b200 import wav

ROOT = Path(__file__).resolve().parent.parent


def rnd(n, c, seed):
    return np.random.default_rng(seed).uniform(-1, 1, (n, c))


def test_float32_roundtrip_bit_exact(tmp_path):  # test_wav.cpp:100-109
    x = rnd(1000, 3, 1).astype(np.float32).astype(np.float64)
    p = tmp_path / "f.wav"
    wav.write_wav(str(p), x, 44100.0, "float32")
    y, fs = wav.read_wav(str(p))
    assert fs == 44100.0 and np.array_equal(x, y)


def test_pcm16_and_pcm24_quantize(tmp_path):  # test_wav.cpp:111-140
    x = rnd(999, 2, 2)
    for fmt, full in (("pcm16", 32768.0), ("pcm24", 8388608.0)):
        p = tmp_path / f"{fmt}.wav"
        wav.write_wav(str(p), x, 48000.0, fmt)
        y, _ = wav.read_wav(str(p))
        assert np.abs(y - x).max() <= 0.5 / full + 1e-15
    p = tmp_path / "neg.wav"
    wav.write_wav(str(p), np.array([[-1.0], [0.999999]]), 48000.0, "pcm24")
    y, _ = wav.read_wav(str(p))
    assert y[0, 0] == -1.0 and y[1, 0] > 0.99


def _craft_pcm16(ch, rate, frames, extensible=False, junk=False):
    fmt = struct.pack("<HHIIHH", 0xFFFE if extensible else 1, ch, rate, rate * 2 * ch, 2 * ch, 16)
    if extensible:
        fmt += struct.pack("<HHI", 22, 16, 0) + struct.pack("<H", 1) + b"\x00" * 14
    body = b"WAVE" + b"fmt " + struct.pack("<I", len(fmt)) + fmt
    if junk:
        body += b"JUNK" + struct.pack("<I", 3) + b"abc\x00"
    data = struct.pack(f"<{len(frames)}h", *frames)
    body += b"data" + struct.pack("<I", len(data)) + data
    return b"RIFF" + struct.pack("<I", len(body)) + body


def test_crafted_files_parse(tmp_path):  # test_wav.cpp:142-158
    for ext in (False, True):
        for junk in (False, True):
            p = tmp_path / f"c{ext}{junk}.wav"
            p.write_bytes(_craft_pcm16(2, 22050, [16384, -16384, 0, 32767], ext, junk))
            y, fs = wav.read_wav(str(p))
            assert fs == 22050 and y.shape == (2, 2)
            assert y[0, 0] == 0.5 and y[0, 1] == -0.5 and y[1, 1] == 32767 / 32768


def test_parse_failures_carry_offsets(tmp_path):  # test_wav.cpp:160-202
    p = tmp_path / "bad.wav"
    p.write_bytes(b"RIFX" + b"\x00" * 8)
    with pytest.raises(wav.WavError) as e:
        wav.read_wav(str(p))
    assert e.value.offset == 0
    p.write_bytes(b"RIFF\x00\x00\x00\x00WAVE" + b"data\x04\x00\x00\x00abcd")
    with pytest.raises(wav.WavError):
        wav.read_wav(str(p))  # data before fmt
    p.write_bytes(_craft_pcm16(1, 8000, [1, 2])[:30])
    with pytest.raises(wav.WavError) as e:
        wav.read_wav(str(p))
    assert e.value.offset > 0
    with pytest.raises(ValueError):
        wav.write_wav(str(tmp_path / "x.wav"), np.zeros((4, 17)))
    # test_wav.cpp:172-180: a valid header, the file shortened by 5 bytes (data shorter than declared)
    p.write_bytes(_craft_pcm16(1, 48000, [1, 2, 3, 4])[:-5])
    with pytest.raises(wav.WavError) as e:
        wav.read_wav(str(p))
    assert e.value.offset > 0
    # test_wav.cpp:182, 199-201, 208: missing file, zero sample rate, unwritable path
    with pytest.raises(wav.WavError):
        wav.read_wav(str(tmp_path / "does_not_exist.wav"))
    p.write_bytes(_craft_pcm16(1, 0, [0]))
    with pytest.raises(wav.WavError):
        wav.read_wav(str(p))
    with pytest.raises(wav.WavError):
        wav.write_wav("/nonexistent_dir/x.wav", np.zeros((4, 1)))


def _cli(*args, env=None):
    return subprocess.run([sys.executable, "-m", "paper_2310_00319_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True, env=env)


def test_cli_usage_error_exit_code():
    assert _cli("process").returncode == 2
    assert _cli("nope").returncode == 2


@pytest.mark.gpu
def test_cli_process_identity_and_flip(tmp_path):
    out = tmp_path / "o.wav"
    r = _cli("process", "--input", "ones:4096", "--ir", "+delta", "--output", str(out), "--block", "512",
             "--ir-len", "2048")
    assert r.returncode == 0, r.stderr
    assert "real-time factor" in r.stdout
    y, fs = wav.read_wav(str(out))
    assert y.shape == (4096, 1) and np.abs(y[256:] - 1.0).max() < 1e-5  # first hop: window ramp-in
    inp = tmp_path / "i.wav"
    x = rnd(3000, 1, 5) * 0.5  # mono input (a 2-channel input needs a 2-channel IR, as in the reference)
    wav.write_wav(str(inp), x, 48000.0)
    r = _cli("process", "--input", str(inp), "--ir", "delta:-0.5:3", "--output", str(out), "--block", "256")
    assert r.returncode == 0, r.stderr
    y, _ = wav.read_wav(str(out))
    ref = np.zeros_like(x)
    ref[3:] = -0.5 * x[:-3]
    assert np.abs(y[: x.shape[0]] - ref).max() < 1e-5


@pytest.mark.gpu
def test_cli_library_error_exit_code(tmp_path):
    r = _cli("process", "--input", "ones:100", "--ir", "+delta", "--output", str(tmp_path / "o.wav"),
             "--block", "24")
    assert r.returncode == 1 and "error" in r.stderr


def test_reference_signal_generators():
    """pink:SEED and synth:azDEG specs (proj/src/signal_gen.cpp:42-107): host generators."""
    from paper_2310_00319_b200 import workload as W

    p = W.gen_pink(1, 4096)
    assert p.shape == (4096,) and 0.01 < np.std(p) < 1.0 and np.array_equal(p, W.gen_pink(1, 4096))
    h = W.synthetic_binaural_ir(90.0, 2048)
    assert h.shape == (2048, 2)
    itd = round(48000 / 1500)  # full lateral displacement
    assert h[2, 0] == 1.0 and h[2 + itd, 1] == pytest.approx(0.25) and h[3:64, 0].max() == 0.0
    assert np.abs(h[64:]).max() < 0.0316
    h0 = W.synthetic_binaural_ir(0.0, 2048)
    assert h0[2, 0] == 1.0 and h0[2, 1] == 1.0
    assert np.array_equal(h0[64:], h[64:])  # the room tail never depends on azimuth


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["tdc", "cf-tdc", "ola", "ols", "wola"])
def test_cli_process_other_algorithms(tmp_path, algo):
    out = tmp_path / "o.wav"
    r = _cli("process", "--algo", algo, "--input", "sine:1000:6000", "--ir", "delta:0.5:2", "--out", str(out),
             "--block", "512", "--ir-len", "512")
    assert r.returncode == 0, r.stderr
    y, _ = wav.read_wav(str(out))
    x = np.sin(2 * np.pi * 1000 / 48000 * np.arange(6000))
    ref = np.zeros(6000)
    ref[2:] = 0.5 * x[:-2]
    assert y.shape[0] >= 6000
    err = np.abs(y[:6000, 0] - ref)
    if algo == "wola":  # only approximate for a delayed tap (test_reference.cpp:108-120)
        assert err.max() < 0.1
    else:
        assert err.max() < 1e-4


@pytest.mark.gpu
def test_cli_switch_and_compare(tmp_path, monkeypatch):
    monkeypatch.setenv("TVOLAP_OUT_DIR", str(tmp_path))
    r = _cli("switch", "--algo", "tvolap", "--switch-ms", "16", "--out-prefix", "sw")
    assert r.returncode == 0, r.stderr
    assert "transition width 256" in r.stdout
    for f in ("sw_output.wav", "sw_metrics.csv", "sw_metrics.json", "sw_transition.csv"):
        assert (tmp_path / f).exists()
    r = _cli("compare", "--frames", "8192", "--out-prefix", "cmp")
    assert r.returncode == 0, r.stderr
    assert "hann:" in r.stdout and "linear:" in r.stdout
    csv = (tmp_path / "cmp_metrics.csv").read_text()
    assert csv.startswith("fade_shape,fade_duration,window_begin,window_end,max_abs_diff,rms_diff,output_rms,diff_db")
    for f in ("cmp_tvolap.wav", "cmp_cftdc_hann.wav", "cmp_diff_linear.wav", "cmp_metrics.json"):
        assert (tmp_path / f).exists()
