"""`python -m paper_2310_00319_b200.cli process ...` — file-to-file GPU convolution
(SURVEY.md §8f row 3), restating the `process` subcommand of proj/tools/tvolap_cli.cpp:143-182:
parse the IR and input specs, fan a mono input out to the IR's channels, stream it through a
FrameAdapter over the GPU engine (arbitrary chunk -> exact hops), drop the stream delay, write
WAV, print the real-time factor. Exit codes as the reference: 0 ok, 1 library error, 2 usage.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

from . import wav
from .tvolap import FrameAdapter, TvolapProcessor


def out_path(name: str) -> str:
    """Relative output paths may be redirected with TVOLAP_OUT_DIR (tvolap_cli.cpp:22-33)."""
    base = os.environ.get("TVOLAP_OUT_DIR")
    if os.path.isabs(name) or not base:
        return name
    os.makedirs(base, exist_ok=True)
    return os.path.join(base, name)


def parse_input(spec: str, frames: int, fs: float):
    """ones[:N] | sine:FREQ[:N] | white:SEED[:N] | a .wav path (tvolap_cli.cpp:43-75)."""
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
    if kind == "white":
        from . import workload as W

        seed = int(parts[1]) if len(parts) > 1 else 1
        n = int(parts[2]) if len(parts) > 2 else frames
        cfg = W.CONFIGS["C1"].scaled(seed=seed)
        return W.white(cfg, 0, 1, 0, n, dtype=np.float64).T, fs
    return wav.read_wav(spec)


def parse_ir(spec: str, ir_len: int, fs: float):
    """+delta | -delta | delta:GAIN[:DELAY] | a .wav path (tvolap_cli.cpp:77-98)."""
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
    return wav.read_wav(spec)


def run_process(args) -> int:
    ir, ir_fs = parse_ir(args.ir, args.ir_len, args.fs)
    x, x_fs = parse_input(args.input, args.frames, ir_fs)
    if x_fs != ir_fs:
        raise ValueError("input and filter sample rates differ")
    if x.shape[1] == 1 and ir.shape[1] > 1:
        x = np.repeat(x, ir.shape[1], axis=1)
    proc = TvolapProcessor(ir, args.block // 2, device=args.device)
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


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="tvolap-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("process", help="convolve an input with an IR on the GPU (tvolap)")
    p.add_argument("--input", required=True)
    p.add_argument("--ir", required=True)
    p.add_argument("--output", required=True)
    p.add_argument("--ir-len", type=int, default=2048)
    p.add_argument("--block", type=int, default=512, help="2L (hop = block / 2)")
    p.add_argument("--frames", type=int, default=48000)
    p.add_argument("--fs", type=float, default=48000.0)
    p.add_argument("--format", default="float32", choices=["pcm16", "pcm24", "float32"])
    p.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    try:
        return run_process(args)
    except (ValueError, RuntimeError, OSError) as e:  # library errors -> 1 (tvolap_cli.cpp:354-383)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
