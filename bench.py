#!/usr/bin/env python
"""Benchmark of the TVOLAP hot path on B200 (BASELINE.json metric).

metric: convolved channel-samples/s. Workload: BASELINE config C2 (configs[1]):
64 independent channels, fp32, L=256, M=64 (IR 32768 taps), each channel
switching to a freshly seeded IR every 16 blocks, 30 s of white noise per
channel = 5625 hops. One step = one full 30 s pass from zero state: the 352
exchange_filter + process_hops(16 hops) drive() loop as one tvolap_process_switching
call on device-resident inputs (run as a time-parallel pass: K4 of all 352 sets,
K1 of all hops, one MAC/inverse CTA per (channel, 16-hop period)).
Multi-GPU (torchrun): one process per GPU, each rank runs its own 64 channels
(lanes rank*64 ..), no data-path collective — weak scaling; time = max over
ranks of CUDA-event time.

Prints ONE JSON line on rank 0. `--impl reference` times the reference
algorithm's CPU path (the fp64 oracle port; the C++ reference itself needs
Eigen and cannot be built here) on the box's host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2310_00319_b200 import workload as W  # noqa: E402

METRIC = "convolved channel-samples/s"
UNIT = "channel-samples/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def config_block(cfg, n_hops, world):
    if cfg.mode == "fresh":
        sw = f"fresh seeded IR per channel every {cfg.period} blocks, T60~U[{cfg.t60[0]},{cfg.t60[1]}] s"
    else:
        sw = (f"bank of {cfg.n_bank} x {cfg.ears}-ear decaying-noise IRs (T60 {cfg.t60[0]} s), "
              + ("alternating every %d blocks" % cfg.period if cfg.n_bank == 2 else "seeded random choice per block"))
    return {
        "workload": f"{cfg.name}: {cfg.sources} source(s) x {cfg.ears} ear(s) per GPU, fp32, L={cfg.hop} "
                    f"(4L={4 * cfg.hop} FFT), M={cfg.partitions} (IR {cfg.ir_length} taps), {sw}, "
                    f"{cfg.seconds:g} s white noise" + (", summed into a stereo mix" if cfg.mix else ""),
        "channels_per_gpu": cfg.lanes,
        "hop": cfg.hop,
        "partitions": cfg.partitions,
        "hops_per_step": n_hops,
        "l2": f"inputs larger than L2: {cfg.sources * n_hops * cfg.hop * 4 / 1e6:.1f} MB input + "
              f"{cfg.lanes * n_hops * cfg.hop * 4 / 1e6:.1f} MB output streamed per step per GPU",
        "parallelism": f"lanes sharded, {world} GPU(s), "
                       + ("NCCL all-reduce of the stereo mix" if cfg.mix and world > 1 else "no collective"),
    }


# ----------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampled every 20 ms from before the warm-up on; a reader thread stamps each line
    on arrival, and stop(t0, t1) summarises the samples that arrived inside the timed region
    (falling back to warm-up + timed region when the region is shorter than the sampling)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        import threading

        self.proc = None
        self.idx = gpu_index
        self.lines = []
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                self.lines.append((time.time(), line))

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    @staticmethod
    def summarise(lines):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, line in lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}

    def stop(self, t0=None, t1=None):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=5)
        lines = list(self.lines)
        if t0 is not None:
            inside = [(t, l) for t, l in lines if t0 <= t <= t1 + 0.03]
            out = self.summarise(inside)
            if out["samples"]:
                out["window"] = "timed region"
                return out
        out = self.summarise(lines)
        out["window"] = "warm-up + timed region (timed region shorter than the 20 ms sampling)"
        return out


# ----------------------------------------------------------------------------- CPU legs
def cpu_sample(cfg, lanes, n_hops, threads, want_output=False):
    """The reference algorithm (fp64 oracle port) over a bounded sample of the workload."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O  # bench's cpu_baseline / reference leg: the checker, never the product

    x = W.white(cfg, 0, lanes, 0, n_hops * cfg.hop, dtype=np.float64)
    n_sw = -(-n_hops // cfg.period)
    irs = np.stack([W.fresh_irs(cfg, k, 0, lanes, dtype=np.float64) for k in range(n_sw)])
    secs, y = O.run_workload(cfg.hop, cfg.partitions, lanes, 1, n_hops, x, 0, fresh_ir=irs, period=cfg.period,
                             want_output=want_output, threads=threads)
    return secs, y


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    threads = W.host_threads()
    lanes, n_hops = cfg.sources, 256
    used = min(threads, lanes)
    vals = []
    for i in range(args.warmup + args.steps):
        secs, _ = cpu_sample(cfg, lanes, n_hops, threads)
        if i >= args.warmup:
            vals.append(lanes * n_hops * cfg.hop / secs)
    v = float(statistics.mean(vals))
    sample = f"{lanes} channels x {n_hops} hops ({n_hops // cfg.period} fresh-IR switches) of {cfg.name} per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * lanes * n_hops * cfg.hop / v, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, n_hops, 1),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": used, "kind": "port", "sample": sample,
                         "note": "fp64 C++ restatement of proj/src/{spectral,partition,engine}.cpp (Eigen "
                                 "unavailable, reference unbuildable); lanes partitioned over std::threads, "
                                 "timed region = process + partition like experiment.cpp:42-52"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--hops", type=int, default=0, help="override hops per step (default: full 30 s)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-hops", type=int, default=512)
    ap.add_argument("--latency-hops", type=int, default=0,
                    help="also time this many single-hop process() calls (pinned host I/O): p50/p99 per-hop latency")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    cfg = W.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg, rank)

    import ctypes

    import torch

    from paper_2310_00319_b200 import _build, shard
    from paper_2310_00319_b200 import tvolap as T
    from paper_2310_00319_b200.tvolap import TvolapBankEngine, TvolapEngine, partition

    _build.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    L, S, M = cfg.hop, cfg.sources, cfg.partitions
    H = args.hops or cfg.hops
    n_sw = -(-H // cfg.period)
    lane0, _ = shard.weak_lanes(S, rank)
    lib = T.lib()

    # ---- inputs resident in HBM (device twins of the seeded generators)
    t0 = time.time()
    x = torch.empty((S, H * L), dtype=torch.float32, device=dev)
    T._check(lib.tvolap_gen_white_device(local, cfg.seed, lane0, S, 0, H * L, ctypes.c_void_p(x.data_ptr()), H * L))
    out = torch.empty((cfg.lanes, H * L), dtype=torch.float32, device=dev)

    def gen_irs(items, dst):
        la = np.array([i[0] for i in items], np.int64)
        ea = np.array([i[1] for i in items], np.int64)
        ka = np.array([i[2] for i in items], np.int64)
        ta = np.array([W.t60_of(cfg, int(l), int(k)) for l, _, k in items], np.float64)
        T._check(lib.tvolap_gen_irs_device(local, cfg.seed, len(items), la.ctypes.data, ea.ctypes.data,
                                           ka.ctypes.data, ta.ctypes.data, W.FS, cfg.ir_length,
                                           ctypes.c_void_p(dst.data_ptr())))

    def fit_block(e):
        """Blocks never span a filter switch, so a block longer than the switch period would
        load each delay-line / filter slice for fewer hops: cap it at the period (C4: 8)."""
        j, _, _ = e.block_config()
        if cfg.period < j:
            e.set_block_config(max(2, 1 << (cfg.period.bit_length() - 1)))

    sched = mix = irs = None
    n_pool = n_sw  # distinct IR sets held in HBM (and pinned host memory for e2e)
    if cfg.mode == "fresh":
        # C4's 704 switches x 256 channels x 131072 taps would not fit: cycle through a pool of
        # distinct seeded sets (<= 24 GB); every switch still uploads + transforms a whole set
        n_pool = int(max(2, min(n_sw, 24e9 // (S * cfg.ir_length * 4))))
        irs = torch.empty((n_pool, S, cfg.ir_length), dtype=torch.float32, device=dev)
        gen_irs([(lane0 + s, 0, k) for k in range(n_pool) for s in range(S)], irs)
        ir0 = W.fresh_irs(cfg, 0, lane0, S)[:, 0, :]
        eng = TvolapEngine(partition(ir0.T, L, M), device=local)
        fit_block(eng)
        distinct = S
    else:
        bank = torch.empty((cfg.n_bank, cfg.ears, cfg.ir_length), dtype=torch.float32, device=dev)
        gen_irs([(b, e, 0) for b in range(cfg.n_bank) for e in range(cfg.ears)], bank)
        sched_h = W.schedule(cfg, 0, H, lane0, S)
        sched = torch.from_numpy(sched_h).to(dev)
        distinct = float(np.mean([np.unique(r).size for r in sched_h[: min(H, 512)]]))
        eng = TvolapBankEngine(bank, L, S, min_partitions=M, device=local)
        if cfg.mix:
            mix = torch.empty((cfg.ears, H * L), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    log(f"[rank {rank}] {cfg.name}: generated {x.numel() * 4 / 1e6:.0f} MB input"
        f"{'' if irs is None else f' + {irs.numel() * 4 / 1e9:.2f} GB IRs'} in {time.time() - t0:.1f} s")
    stream = torch.cuda.Stream(device=dev)
    eng.set_stream(stream.cuda_stream)
    P, NT = eng.launch_config()
    log(f"[rank {rank}] launch config: {P} CTAs/channel (cluster), {NT} threads/CTA")

    def step(e, xs, outs, ir_set, sch):
        e.reset()
        if cfg.mode == "fresh":
            # the drive() loop (exchange before every period's hops) as one call:
            # device-resident -> the time-parallel pass (few channels) or one hop-blocked launch with
            # in-kernel K4; pinned host buffers -> the chunked H2D / launch / D2H pipeline
            e.process_switching(xs, [ir_set[k % n_pool] for k in range(n_sw)], cfg.period, out=outs)
        else:
            e.process_hops(xs, out=outs, schedule=sch)
            if mix is not None and outs.is_cuda:
                T._check(lib.tvolap_mix_device(local, S, cfg.ears, H * L, ctypes.c_void_p(outs.data_ptr()), H * L,
                                               ctypes.c_void_p(mix.data_ptr()), H * L,
                                               ctypes.c_void_p(stream.cuda_stream)))
                if world > 1:
                    with torch.cuda.stream(stream):
                        shard.mix_allreduce(mix)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(local)
    for _ in range(args.warmup):
        step(eng, x, out, irs, sched)
    barrier()
    launches0 = eng.kernel_launches()
    wide0 = eng.wide_passes() if hasattr(eng, "wide_passes") else 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start = time.time()
    ev0.record(stream)
    for _ in range(args.steps):
        step(eng, x, out, irs, sched)
    ev1.record(stream)
    barrier()
    t_end = time.time()
    clk = clocks.stop(t_start, t_end)
    elapsed = ev0.elapsed_time(ev1)
    gpu_launches = eng.kernel_launches() - launches0 + (args.steps if mix is not None else 0)
    wide = (eng.wide_passes() - wide0 if hasattr(eng, "wide_passes") else 0) > 0
    # Per-launch kernel durations: a second pass of the same steps with CUDA events around every
    # hop launch on the engine stream. Timing events serialise the programmatic-dependent-launch
    # chain (K4 -> hop launch overlap), so they stay out of the timed region above.
    prof_steps = max(1, min(args.steps, 3))
    eng.set_profiling(True)
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    for _ in range(prof_steps):
        step(eng, x, out, irs, sched)
    ev3.record(stream)
    barrier()
    kern_ms, kern_n = eng.kernel_time()
    eng.set_profiling(False)
    prof_elapsed = ev2.elapsed_time(ev3)
    elapsed = shard.max_over_ranks(elapsed, dev)
    ms_per_step = elapsed / args.steps
    samples_per_step = world * cfg.lanes * H * L
    value = samples_per_step / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel (fused hop kernel), algorithmic bytes per launch
    pk = peaks()
    hbm = pk.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    if not hbm:
        hbm, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    hops_per_launch = H * prof_steps / kern_n if kern_n else H
    bytes_hop = W.bytes_per_hop(cfg, distinct_filters=distinct)
    bytes_launch = bytes_hop * hops_per_launch
    avg_launch_ms = kern_ms / kern_n if kern_n else float("nan")
    achieved = bytes_launch / (avg_launch_ms / 1e3) / 1e9
    traffic = None
    ncu_view = None
    summ = ROOT / "profiles" / f"ncu_summary_{cfg.name}.json"
    if summ.exists():
        try:
            sj = json.loads(summ.read_text())
            # per hop when the capture records it (its launch length may differ from this run's)
            traffic = sj["dram_bytes_per_hop"] * hops_per_launch if sj.get("dram_bytes_per_hop") \
                else sj.get("dram_bytes_per_launch")
            # what actually bounds the captured kernel (committed capture, cold caches)
            k = next((l for l in sj.get("per_launch", []) if "wide_mac" in l.get("name", "")),
                     (sj.get("per_launch") or [{}])[0])
            us = k.get("gpu__time_duration.sum")
            dram = (k.get("dram__bytes_read.sum") or 0) + (k.get("dram__bytes_write.sum") or 0)
            ncu_view = {"kernel": k.get("name", "")[:60], "source": f"profiles/{summ.name}",
                        "dram_gbs": dram / (us * 1e-6) / 1e9 if us else None,
                        "dram_frac": dram / (us * 1e-6) / 1e9 / hbm if us else None,
                        "fma_pipe_pct": k.get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                        "warps_active_pct": k.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                        "top_stalls": k.get("top_stalls")}
        except Exception:
            traffic = None
    if wide:  # time-parallel pass: the MAC/inverse launch dominates; K4 and K1 are separate launches
        kname = (f"wide_mac_kernel (K4 of the tile's filter set into an L2 scratch slot + K3 + K5 + OLA, one CTA "
                 f"per (channel, filter period <= 16 hops)), {hops_per_launch:g} hops x {S} sources per launch; K1 of "
                 "all hops (wide_forward_kernel, ~13% of the step) is a separate launch outside this kernel's time")
    else:
        kname = (f"tvolap_block_kernel (K1-K5 fused{', K4 for the next switch in the barrier gaps' if cfg.mode == 'fresh' else ''}), "
                 f"{hops_per_launch:g} hops x {S} sources per launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "peak_source": peak_src,
                "kernel": kname,
                "pass_achieved": bytes_hop * H / (ms_per_step / 1e3) / 1e9,
                "ncu": ncu_view,
                "avg_launch_ms": avg_launch_ms, "launches": kern_n, "bytes_per_hop": bytes_hop,
                "bytes_per_launch": bytes_launch, "distinct_filters_per_hop": distinct,
                "kernel_share_of_step": kern_ms / prof_elapsed if prof_elapsed else None,
                "timing": f"avg launch from a separate event-instrumented pass of {prof_steps} step(s) "
                          "(share = kernel time / that pass's elapsed)"}
    if wide:
        roofline["note"] = ("algorithmic bytes (SURVEY 8d: every output re-reads M delay-line spectra and M filter "
                            "spectra) over the MAC launch's time; the kernel reads each spectrum once per 16-hop tile, "
                            "so frac can exceed 1; pass_achieved = the same bytes over the whole step (all launches)")
    elif cfg.name in ("C1", "C2"):
        roofline["note"] = "delay line + filter pool are L2-resident in this config, so frac vs HBM can exceed 1"

    # ---- e2e through the public API with pinned host buffers (H2D inputs [+ IRs], D2H outputs)
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        oh = torch.empty(tuple(out.shape), dtype=torch.float32, pin_memory=True)
        h2d = xh.numel() * 4
        if cfg.mode == "fresh":
            irh = torch.empty(irs.shape, dtype=torch.float32, pin_memory=True)
            irh.copy_(irs)
            eng2 = TvolapEngine(partition(ir0.T, L, M), device=local)
            fit_block(eng2)
            h2d += n_sw * S * cfg.ir_length * 4  # one whole set uploaded per switch
            schh = None
        else:
            irh = None
            schh = sched.cpu().pin_memory()
            h2d += schh.numel() * 4
            eng2 = TvolapBankEngine(bank, L, S, min_partitions=M, device=local)
        eng2.set_host_async(True)
        step(eng2, xh, oh, irh, schh)
        eng2.synchronize()
        barrier()
        tw = time.perf_counter()
        for _ in range(args.steps):
            step(eng2, xh, oh, irh, schh)
            eng2.synchronize()
        barrier()
        e2e_s = (time.perf_counter() - tw) / args.steps
        e2e_s = shard.max_over_ranks(e2e_s, dev)
        same = bool(torch.equal(oh, out.cpu()))
        e2e = {"value": samples_per_step / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(oh.numel() * 4), "ms_per_step": e2e_s * 1e3,
               "timing": "host wall clock around each full pass incl. final synchronize",
               "matches_device_path": same}
        del irh

    latency = None
    if args.latency_hops:
        lat_eng = (TvolapBankEngine(bank, L, S, min_partitions=M, device=local) if cfg.mode == "bank"
                   else TvolapEngine(partition(ir0.T, L, M), device=local))
        lat_eng.set_stream(stream.cuda_stream)
        xin = torch.empty((S, L), dtype=torch.float32, pin_memory=True)
        yout = torch.empty((cfg.lanes, L), dtype=torch.float32, pin_memory=True)
        xsrc = x[:, : (args.latency_hops + 8) * L].cpu()
        sch_np = sched.cpu().numpy() if sched is not None else None
        gpu_ms, host_ms = [], []
        for h in range(args.latency_hops + 8):
            xin.copy_(xsrc[:, h * L:(h + 1) * L])
            if sch_np is not None:
                lat_eng.select_bank(sch_np[h])
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0h = time.perf_counter()
            a.record(stream)
            T._check(lib.tvolap_process(lat_eng._h, ctypes.c_void_p(xin.data_ptr()), L, L, S,
                                        ctypes.c_void_p(yout.data_ptr()), L))
            b.record(stream)
            b.synchronize()
            if h >= 8:
                host_ms.append((time.perf_counter() - t0h) * 1e3)
                gpu_ms.append(a.elapsed_time(b))
        q = lambda v, p: float(np.percentile(v, p))  # noqa: E731
        latency = {"hops": args.latency_hops, "gpu_ms_p50": q(gpu_ms, 50), "gpu_ms_p99": q(gpu_ms, 99),
                   "host_ms_p50": q(host_ms, 50), "host_ms_p99": q(host_ms, 99),
                   "hop_period_ms": 1e3 * L / W.FS,
                   "what": "one process() call per hop: pinned H2D of the hop, fused kernel, D2H of the outputs; "
                           "CUDA events on the engine stream (gpu) and host wall clock (host)"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded white noise + decaying-noise IRs generated on device)",
        "config": config_block(cfg, H, world), "clocks": clk, "gpu_launches": int(gpu_launches),
        "roofline": roofline, "e2e": e2e, "latency": latency,
        "realtime_factor": (H * L / W.FS) / (ms_per_step / 1e3),
    }
    if cfg.mode == "fresh" and n_pool < n_sw:
        line["config"]["ir_sets"] = (f"{n_sw} switches per step cycle through {n_pool} distinct seeded IR sets "
                                     "held in HBM (every switch uploads and transforms a whole set)")

    # ---- CPU baseline (rank 0, N=1 only): the reference algorithm on host cores, bounded sample
    if rank == 0 and world == 1 and not args.no_cpu and cfg.mode == "fresh":
        threads = W.host_threads()
        ch = min(args.cpu_hops, H)
        secs, yref = cpu_sample(cfg, S, ch, threads, want_output=True)
        y = out[:, : ch * L].double().cpu().numpy()
        rel = float(np.abs(y - yref).max() / np.abs(yref).max())
        secs1, _ = cpu_sample(cfg, 4, 64, 1)
        line["cpu_baseline"] = {
            "value": S * ch * L / secs, "unit": UNIT, "cores": min(threads, S), "kind": "port",
            "sample": f"{S} channels x {ch} hops ({ch // cfg.period} fresh-IR switches) of {cfg.name}",
            "single_thread_value": 4 * 64 * L / secs1,
            "parity_rel_err_vs_gpu": rel,
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
