"""`python -m paper_2310_00319_b200.cli {process,switch,compare} ...` — the reference CLI's
convolution subcommands on the GPU, restating proj/tools/tvolap_cli.cpp:
* process (:143-182): parse the IR and input specs, fan a mono input out to the IR's channels,
  stream it through a FrameAdapter over the chosen GPU processor (--algo tvolap | tdc | cf-tdc |
  ola | ols | wola), drop the stream delay, write WAV, print the real-time factor;
* switch (:184-220): one filter exchange, output WAV + metrics CSV/JSON + transition CSV;
* compare (:222-268): partitioned engine vs crossfaded direct form, WAVs + metrics tables.
Exit codes as the reference: 0 ok, 1 library error, 2 usage.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

from . import experiment as X
from . import wav
from . import workload as W
from .tvolap import CrossfadeConfig, FrameAdapter, make_processor


def out_path(name: str) -> str:
    """Relative output paths may be redirected with TVOLAP_OUT_DIR (tvolap_cli.cpp:22-33)."""
    base = os.environ.get("TVOLAP_OUT_DIR")
    if os.path.isabs(name) or not base:
        return name
    os.makedirs(base, exist_ok=True)
    return os.path.join(base, name)


def write_text(name: str, text: str) -> None:
    with open(out_path(name), "w") as f:
        f.write(text)


def hop_for(algo: str, block: int) -> int:
    """tvolap_cli.cpp:100-104: the partitioned engine hops by block / 2, the others by block."""
    return block // 2 if algo == "tvolap" else block


def parse_input(spec: str, frames: int, fs: float):
    """ones[:N] | sine:FREQ[:N] | pink[:SEED[:N]] | white:SEED[:N] | a .wav path (tvolap_cli.cpp:43-75)."""
    parts = spec.split(":")
    kind = parts[0]
    if kind == "ones":
        n = int(parts[1]) if len(parts) > 1 else frames
        return np.ones((n, 1)), fs
    if kind == "sine":
        freq = float(parts[1]) if len(parts) > 1 else 750.0
        n = int(parts[2]) if len(parts) > 2 else frames
        if not 0 < freq < fs / 2:
            raise ValueError("gen_sine: frequency must lie in (0, f_s/2)")
        return np.sin(2 * np.pi * freq / fs * np.arange(n))[:, None], fs
    if kind == "pink":
        seed = int(parts[1]) if len(parts) > 1 else 1
        n = int(parts[2]) if len(parts) > 2 else frames
        return W.gen_pink(seed, n)[:, None], fs
    if kind == "white":
        seed = int(parts[1]) if len(parts) > 1 else 1
        n = int(parts[2]) if len(parts) > 2 else frames
        cfg = W.CONFIGS["C1"].scaled(seed=seed)
        return W.white(cfg, 0, 1, 0, n, dtype=np.float64).T, fs
    return wav.read_wav(spec)


def parse_ir(spec: str, ir_len: int, fs: float):
    """+delta | -delta | delta:GAIN[:DELAY] | synth:azDEG | a .wav path (tvolap_cli.cpp:77-98)."""
    if spec in ("+delta", "-delta") or spec.startswith("delta:"):
        gain, delay = (1.0 if spec == "+delta" else -1.0), 0
        if spec.startswith("delta:"):
            g, _, d = spec[6:].partition(":")
            gain, delay = float(g), int(d) if d else 0
        if not 0 <= delay < ir_len:
            raise ValueError("delta_ir: delay outside the response")
        h = np.zeros((ir_len, 1))
        h[delay, 0] = gain
        return h, fs
    if spec.startswith("synth:az"):
        return W.synthetic_binaural_ir(float(spec[8:]), ir_len, fs), fs
    return wav.read_wav(spec)


def run_process(args) -> int:
    ir, ir_fs = parse_ir(args.ir, args.ir_len, args.fs)
    x, x_fs = parse_input(args.input, args.frames, ir_fs)
    if x_fs != ir_fs:
        raise ValueError("input and filter sample rates differ")
    if x.shape[1] == 1 and ir.shape[1] > 1:
        x = np.repeat(x, ir.shape[1], axis=1)
    proc = make_processor(args.algo, ir, hop_for(args.algo, args.block), device=args.device)
    adapter = FrameAdapter(proc)
    hop, delay = proc.hop(), proc.stream_delay()
    n_padded = -(-x.shape[0] // hop) * hop
    t0 = time.perf_counter()
    head = adapter.push(x)
    pad = adapter.push(np.zeros((n_padded - x.shape[0] + delay, x.shape[1])))
    tail = adapter.flush()
    seconds = time.perf_counter() - t0
    stream = np.concatenate([head, pad, tail])
    y = stream[delay: delay + n_padded]
    path = out_path(args.output)
    wav.write_wav(path, y, x_fs, args.format)
    print(f"wrote {path} ({y.shape[0]} frames)")
    print(f"real-time factor: {(x.shape[0] / x_fs) / seconds if seconds > 0 else 0.0}")
    return 0


def run_switch_cmd(args) -> int:
    """tvolap_cli.cpp:184-220."""
    ir_a, fs = parse_ir(args.ir_a, args.ir_len, args.fs)
    ir_b, _ = parse_ir(args.ir_b, args.ir_len, args.fs)
    x, x_fs = parse_input(args.input, args.frames, fs)
    hop = hop_for(args.algo, args.block)
    sample = int(round(args.switch_ms / 1000.0 * x_fs))
    fade = CrossfadeConfig(args.fade_duration if args.fade_duration > 0 else hop,
                           CrossfadeConfig.LINEAR if args.fade_shape == "linear" else CrossfadeConfig.HANN)
    run = X.run_switch(x, ir_a, ir_b, hop, sample, args.algo, x_fs, fs, fs, device=args.device, fade=fade)
    wav.write_wav(out_path(args.out_prefix + "_output.wav"), run.output, x_fs, args.format)
    write_text(args.out_prefix + "_metrics.csv", X.metrics_csv([run.metrics]))
    write_text(args.out_prefix + "_metrics.json", X.metrics_json([run.metrics]))
    write_text(args.out_prefix + "_transition.csv", X.transition_csv(run, run.metrics.hop, 3 * run.metrics.hop))
    secs = (x.shape[0] / x_fs)
    print(f"switch applied at sample {run.metrics.switch_boundary}, transition width {run.metrics.transition_width}")
    print(f"real-time factor: {secs / run.engine_seconds if run.engine_seconds > 0 else 0.0}")
    return 0


def run_compare_cmd(args) -> int:
    """tvolap_cli.cpp:222-268."""
    ir_a, fs = parse_ir(args.ir_a, args.ir_len, args.fs)
    ir_b, _ = parse_ir(args.ir_b, args.ir_len, args.fs)
    x, x_fs = parse_input(args.input, args.frames, fs)
    hop = args.block // 2
    sample = int(round(args.switch_ms / 1000.0 * x_fs))
    shapes = {"hann": [CrossfadeConfig.HANN], "linear": [CrossfadeConfig.LINEAR]}.get(
        args.shape, [CrossfadeConfig.HANN, CrossfadeConfig.LINEAR])
    rows, wrote = [], False
    for sh in shapes:
        run = X.run_compare(x, ir_a, ir_b, hop, sample, sh, device=args.device)
        if not wrote:
            wav.write_wav(out_path(args.out_prefix + "_tvolap.wav"), run.tvolap.output, x_fs, args.format)
            wrote = True
        name = run.metrics.fade_shape
        wav.write_wav(out_path(f"{args.out_prefix}_cftdc_{name}.wav"), run.crossfaded.output, x_fs, args.format)
        wav.write_wav(out_path(f"{args.out_prefix}_diff_{name}.wav"), run.difference, x_fs, args.format)
        print(f"{name}: max |diff| {run.metrics.max_abs_diff}, rms diff {run.metrics.diff_db} dB re output")
        rows.append(run.metrics)
    write_text(args.out_prefix + "_metrics.csv", X.compare_csv(rows))
    write_text(args.out_prefix + "_metrics.json", X.compare_json(rows))
    return 0


ALGOS = ["tvolap", "tdc", "cf-tdc", "ola", "ols", "wola"]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="tvolap-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("process", help="time-invariant filtering of a signal on the GPU")
    p.add_argument("--algo", default="tvolap", choices=ALGOS)
    p.add_argument("--input", required=True)
    p.add_argument("--ir", required=True)
    p.add_argument("--output", "--out", dest="output", required=True)
    p.add_argument("--ir-len", type=int, default=2048)
    p.add_argument("--block", type=int, default=512, help="stepping block (2L for tvolap)")
    p.add_argument("--frames", type=int, default=16384)
    p.add_argument("--fs", type=float, default=48000.0)
    p.add_argument("--format", default="float32", choices=["pcm16", "pcm24", "float32"])
    p.add_argument("--device", type=int, default=0)
    s = sub.add_parser("switch", help="single filter-exchange experiment")
    s.add_argument("--algo", default="tvolap", choices=ALGOS)
    s.add_argument("--input", default="ones")
    s.add_argument("--ir-a", default="+delta")
    s.add_argument("--ir-b", default="-delta")
    s.add_argument("--ir-len", type=int, default=2048)
    s.add_argument("--block", type=int, default=512)
    s.add_argument("--frames", type=int, default=16384)
    s.add_argument("--fs", type=float, default=48000.0)
    s.add_argument("--switch-ms", type=float, default=3.0)
    s.add_argument("--fade-duration", type=int, default=0, help="cf-tdc fade length (0: one hop)")
    s.add_argument("--fade-shape", default="hann", choices=["hann", "linear"])
    s.add_argument("--out-prefix", default="switch")
    s.add_argument("--format", default="float32", choices=["pcm16", "pcm24", "float32"])
    s.add_argument("--device", type=int, default=0)
    c = sub.add_parser("compare", help="partitioned engine vs crossfaded direct convolution")
    c.add_argument("--input", default="pink:1")
    c.add_argument("--ir-a", default="synth:az0")
    c.add_argument("--ir-b", default="synth:az90")
    c.add_argument("--ir-len", type=int, default=2048)
    c.add_argument("--block", type=int, default=512)
    c.add_argument("--frames", type=int, default=16384)
    c.add_argument("--fs", type=float, default=48000.0)
    c.add_argument("--switch-ms", type=float, default=7.0)
    c.add_argument("--shape", default="both", choices=["hann", "linear", "both"])
    c.add_argument("--out-prefix", default="compare")
    c.add_argument("--format", default="float32", choices=["pcm16", "pcm24", "float32"])
    c.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    try:
        if args.cmd == "switch":
            return run_switch_cmd(args)
        if args.cmd == "compare":
            return run_compare_cmd(args)
        return run_process(args)
    except (ValueError, RuntimeError, OSError) as e:  # library errors -> 1 (tvolap_cli.cpp:354-383)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
