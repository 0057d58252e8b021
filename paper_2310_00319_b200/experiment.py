"""Switch / compare experiments and metric tables over the GPU processors.

Restates proj/src/experiment.cpp:23-161 (make_proc, drive, run_switch, run_compare) and
:163-264 (metrics_csv, metrics_json, compare_csv, compare_json, transition_csv) for every
algorithm of make_processor ("tvolap" on the B200 engine; "tdc", "cf-tdc", "ola", "ols", "wola"
on the GPU comparison convolvers), so the reference's switching analysis (transition start /
width / click steps, engine vs crossfade difference) runs on GPU output. The three runs
(switched, old filter throughout, new filter throughout) use multi-hop calls, which equal one
process() per hop, so outputs before the boundary and after settling match the references to
within fp32 rounding; the detection threshold is 1e-6 of the signal scale (the reference's fp64
engine uses 1e-9).
"""
from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field
from typing import List, Optional

import numpy as np

from .tvolap import (CfTdcProcessor, CrossfadeConfig, IncompatibleFilterError,  # noqa: F401
                     InvalidConfigurationError, InvalidInputError, TvolapProcessor, make_processor)


@dataclass
class SwitchMetrics:
    """experiment.hpp:16-27 — all positions input-aligned (stream delay removed)."""

    algorithm: str = "tvolap"
    hop: int = 0
    audio_latency: int = 0
    stream_delay: int = 0
    switching_latency: int = 0
    switch_boundary: int = 0
    transition_start: int = -1
    transition_width: int = 0
    max_step_transition: float = 0.0
    max_step_steady: float = 0.0


@dataclass
class SwitchRun:
    output: np.ndarray = field(repr=False, default=None)
    old_ref: np.ndarray = field(repr=False, default=None)
    new_ref: np.ndarray = field(repr=False, default=None)
    metrics: SwitchMetrics = field(default_factory=SwitchMetrics)
    engine_seconds: float = 0.0


def _as_frames(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    return a[:, None] if a.ndim == 1 else a


def _make_proc(algorithm: str, ir, hop: int, fade: Optional[CrossfadeConfig], device: int):
    """experiment.cpp:23-29."""
    if algorithm == "cf-tdc" and fade is not None:
        return CfTdcProcessor(ir, hop, fade, device=device)
    return make_processor(algorithm, ir, hop, device=device)


def _drive(proc, padded: np.ndarray, ir_b, switch_call: int) -> np.ndarray:
    """experiment.cpp:33-54: hops in order (plus delay/hop zero hops), filter staged right before
    `switch_call` (negative: never); returns the input-aligned stream."""
    hop, delay = proc.hop(), proc.stream_delay()
    calls = padded.shape[0] // hop + delay // hop
    x = np.zeros((calls * hop, padded.shape[1]), dtype=np.float32)
    x[: padded.shape[0]] = padded
    run = proc.engine().process_hops if isinstance(proc, TvolapProcessor) else proc.process_hops
    lanes = np.ascontiguousarray(x.T)
    cut = switch_call * hop if 0 <= switch_call < calls else calls * hop
    parts = []
    if cut > 0:
        parts.append(run(np.ascontiguousarray(lanes[:, :cut])))
    if cut < calls * hop:
        proc.set_filter(ir_b)
        parts.append(run(np.ascontiguousarray(lanes[:, cut:])))
    stream = np.concatenate(parts, axis=1).T
    return stream[delay: delay + padded.shape[0]].astype(np.float64)


def run_switch(input, ir_a, ir_b, hop: int, requested_switch_sample: int, algorithm: str = "tvolap",
               input_rate: float = 48000.0, ir_a_rate: float = 48000.0, ir_b_rate: float = 48000.0,
               device: int = 0, fade: Optional[CrossfadeConfig] = None) -> SwitchRun:
    """run_switch (experiment.cpp:58-128) on the GPU processors."""
    import time

    x = _as_frames(input)
    a, b = _as_frames(ir_a), _as_frames(ir_b)
    if x.shape[0] < 1:
        raise InvalidInputError("run_switch: empty input")
    if not (input_rate == ir_a_rate == ir_b_rate):
        raise InvalidConfigurationError("run_switch: input and filters must share a sample rate")
    if x.shape[1] == 1 and a.shape[1] > 1:  # fan_out (audio_buffer.hpp:60-67)
        x = np.repeat(x, a.shape[1], axis=1)

    proc = _make_proc(algorithm, a, hop, fade, device)
    ref_old = _make_proc(algorithm, a, hop, fade, device)
    ref_new = _make_proc(algorithm, b, hop, fade, device)
    h = proc.hop()
    calls_in = -(-x.shape[0] // h)
    n = calls_in * h
    if requested_switch_sample < 0 or requested_switch_sample >= x.shape[0]:
        raise InvalidConfigurationError("run_switch: switch sample outside the signal")
    boundary = ((requested_switch_sample + h // 2) // h) * h
    boundary = min(boundary, (calls_in - 1) * h)
    padded = np.zeros((n, x.shape[1]))
    padded[: x.shape[0]] = x

    if algorithm == "tvolap" and -(-b.shape[0] // (2 * h)) > proc.engine().partition_count():
        raise IncompatibleFilterError("replacement filter partition count differs")
    run = SwitchRun()
    switch_call = boundary // h + proc.stream_delay() // h
    t0 = time.perf_counter()
    run.output = _drive(proc, padded, b, switch_call)
    run.engine_seconds = time.perf_counter() - t0
    run.old_ref = _drive(ref_old, padded, None, -1)
    run.new_ref = _drive(ref_new, padded, None, -1)

    m = run.metrics
    m.algorithm, m.hop = algorithm, h
    m.audio_latency, m.stream_delay = proc.latency(), proc.stream_delay()
    m.switching_latency, m.switch_boundary = proc.switching_latency(), boundary
    scale = max(np.abs(run.old_ref).max(), np.abs(run.new_ref).max(), np.finfo(float).tiny)
    tol = 1e-6 * scale  # the reference's 1e-9 is an fp64 threshold; fp32 rounding sits ~1e-7
    dev_old = np.abs(run.output - run.old_ref).max(axis=1) > tol
    m.transition_start = int(np.argmax(dev_old)) if dev_old.any() else -1
    dev_new = np.abs(run.output - run.new_ref).max(axis=1) > tol
    late = np.nonzero(dev_new[boundary:])[0]
    settled = boundary + int(late[-1]) + 1 if late.size else boundary
    m.transition_width = settled - boundary
    steps = np.abs(np.diff(run.output, axis=0)).max(axis=1)  # step at t (t >= 1)
    t = np.arange(1, n)
    inside = (t >= boundary) & (t <= settled)
    m.max_step_transition = float(steps[inside].max()) if inside.any() else 0.0
    m.max_step_steady = float(steps[~inside].max()) if (~inside).any() else 0.0
    return run


@dataclass
class CompareMetrics:
    """experiment.hpp:47-56."""

    fade_shape: str = "hann"
    fade_duration: int = 0
    window_begin: int = 0
    window_end: int = 0
    max_abs_diff: float = 0.0
    rms_diff: float = 0.0
    output_rms: float = 0.0
    diff_db: float = 0.0


@dataclass
class CompareRun:
    tvolap: SwitchRun = None
    crossfaded: SwitchRun = None
    difference: np.ndarray = field(repr=False, default=None)
    metrics: CompareMetrics = field(default_factory=CompareMetrics)


def run_compare(input, ir_a, ir_b, hop: int, requested_switch_sample: int, shape: int = CrossfadeConfig.HANN,
                device: int = 0) -> CompareRun:
    """run_compare (experiment.cpp:130-161): the partitioned engine against the crossfaded direct
    form (fade duration = hop), both on the GPU."""
    fade = CrossfadeConfig(hop, shape)
    run = CompareRun()
    run.tvolap = run_switch(input, ir_a, ir_b, hop, requested_switch_sample, "tvolap", device=device)
    run.crossfaded = run_switch(input, ir_a, ir_b, hop, requested_switch_sample, "cf-tdc", device=device, fade=fade)
    run.difference = run.tvolap.output - run.crossfaded.output
    m = run.metrics
    m.fade_shape = "linear" if shape == CrossfadeConfig.LINEAR else "hann"
    m.fade_duration = fade.duration
    n = run.difference.shape[0]
    b = run.tvolap.metrics.switch_boundary
    m.window_begin, m.window_end = b, min(n, b + 3 * hop)
    m.max_abs_diff = float(np.abs(run.difference).max())
    win = run.difference[m.window_begin:m.window_end]
    out = run.tvolap.output[m.window_begin:m.window_end]
    m.rms_diff = float(np.sqrt(np.mean(win ** 2)))
    m.output_rms = float(np.sqrt(np.mean(out ** 2)))
    m.diff_db = float(20.0 * np.log10(max(m.rms_diff, 1e-300) / max(m.output_rms, 1e-300)))
    return run


def _fmt(v: float) -> str:
    return "%.12g" % v


def metrics_csv(rows: List[SwitchMetrics]) -> str:
    """experiment.cpp:163-181."""
    out = ("algorithm,hop,audio_latency,stream_delay,switching_latency,switch_boundary,"
           "transition_start,transition_width,max_step_transition,max_step_steady\n")
    for m in rows:
        out += ",".join([m.algorithm, str(m.hop), str(m.audio_latency), str(m.stream_delay),
                         str(m.switching_latency), str(m.switch_boundary), str(m.transition_start),
                         str(m.transition_width), _fmt(m.max_step_transition), _fmt(m.max_step_steady)]) + "\n"
    return out


def metrics_json(rows: List[SwitchMetrics]) -> str:
    """experiment.cpp:183-200."""
    return json.dumps([asdict(m) for m in rows], indent=2) + "\n"


def compare_csv(rows: List[CompareMetrics]) -> str:
    """experiment.cpp:202-218."""
    out = "fade_shape,fade_duration,window_begin,window_end,max_abs_diff,rms_diff,output_rms,diff_db\n"
    for m in rows:
        out += ",".join([m.fade_shape, str(m.fade_duration), str(m.window_begin), str(m.window_end),
                         _fmt(m.max_abs_diff), _fmt(m.rms_diff), _fmt(m.output_rms), _fmt(m.diff_db)]) + "\n"
    return out


def compare_json(rows: List[CompareMetrics]) -> str:
    """experiment.cpp:220-234."""
    return json.dumps([asdict(m) for m in rows], indent=2) + "\n"


def transition_csv(run: SwitchRun, before: int, after: int) -> str:
    """experiment.cpp:236-262: samples around the boundary for plotting."""
    n, ch = run.output.shape
    b = run.metrics.switch_boundary
    lo, hi = max(0, b - before), min(n, b + after)
    head = ["offset"] + [f"output_{c}" for c in range(ch)] + [f"old_ref_{c}" for c in range(ch)] + \
           [f"new_ref_{c}" for c in range(ch)]
    lines = [",".join(head)]
    for t in range(lo, hi):
        vals = [str(t - b)] + [_fmt(v) for v in run.output[t]] + [_fmt(v) for v in run.old_ref[t]] + \
               [_fmt(v) for v in run.new_ref[t]]
        lines.append(",".join(vals))
    return "\n".join(lines) + "\n"
