#!/usr/bin/env python
"""Benchmark of the TVOLAP hot path on B200 (BASELINE.json metric).

metric: convolved channel-samples/s (lanes x hops x L / time), at 1/2/4/8 GPUs, next to the
reference's CPU path on the box's host cores.

Default workload: BASELINE config C5 (configs[4]) — the largest single-GPU config: 4096
channels, fp32, L=32 (4L=128 FFT), M=512 partitions (IR 32768 taps), every channel picking a
seeded-random entry of a 1024-IR bank (T60 0.4 s) every block, 10 s of white noise = 15000 hops.
One step = one full 10-s pass from zero state: tvolap_process_hops with the per-hop bank schedule
on device-resident inputs (run as bank passes: K1 of every hop, the MAC over (tile, channel,
partition group) CTAs, K5 + overlap-add per (tile, channel)). `--config C1..C4` runs the others.

Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run, one process per GPU, NCCL);
channels are sharded across ranks (`--scaling strong`, default: the config's channels split N
ways; `weak`: every rank runs a whole config). No data-path collective except C3's stereo mix,
reduced with NCCL (tvolap_mix_allreduce). Time = max over ranks of CUDA-event time.

JSON line keys beyond the base contract:
  roofline   measured sides of the dominant kernel: HBM (ncu DRAM bytes), L2 (ncu L2->SM bytes)
             and FP32 (reference cost model flops), each over the live per-launch time; `bound`
             names the binding side; the SURVEY §8(d) algorithmic bytes are reported separately
  latency    p50/p99 per-hop GPU latency of the streaming process() API (one hop per call)
  cpu_baseline / parity   the reference (oracle/_ref: the reference's own engine sources) on a
             bounded sample of the same workload on all host cores, and max|y_gpu - y_ref| /
             max|y_ref| of the bench's own outputs on that sample
`--impl reference` times the same sample on the reference's CPU path (rank 0 only).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
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
DEFAULT_CONFIG = "C5"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    out = {}
    for f in (ROOT / "MEASURED_PEAKS.json", ROOT / "profiles" / "l2_peak.json"):
        try:
            out.update(json.loads(f.read_text()))
        except Exception:
            pass
    return out


def config_block(cfg, n_hops, world, lanes_per_rank, scaling):
    if cfg.mode == "fresh":
        sw = f"fresh seeded IR per channel every {cfg.period} blocks, T60~U[{cfg.t60[0]},{cfg.t60[1]}] s"
    else:
        sw = (f"bank of {cfg.n_bank} x {cfg.ears}-ear decaying-noise IRs (T60 {cfg.t60[0]} s), "
              + ("alternating every %d blocks" % cfg.period if cfg.n_bank == 2 else "seeded random choice per block"))
    total = cfg.sources * (world if scaling == "weak" else 1)
    return {
        "workload": f"{cfg.name}: {total} source(s) x {cfg.ears} ear(s), fp32, L={cfg.hop} "
                    f"(4L={4 * cfg.hop} FFT), M={cfg.partitions} (IR {cfg.ir_length} taps), {sw}, "
                    f"{cfg.seconds:g} s white noise" + (", summed into a stereo mix" if cfg.mix else ""),
        "channels_total": total * cfg.ears,
        "sources_per_gpu": lanes_per_rank,
        "hop": cfg.hop,
        "partitions": cfg.partitions,
        "hops_per_step": n_hops,
        "l2": f"inputs larger than L2: {total * n_hops * cfg.hop * 4 / 1e6:.0f} MB input + "
              f"{total * cfg.ears * n_hops * cfg.hop * 4 / 1e6:.0f} MB output per step",
        "parallelism": f"{scaling} channel sharding over {world} GPU(s), "
                       + ("cross-GPU stereo mix (see mix_path)" if cfg.mix and world > 1 else "no collective"),
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
def cpu_sample_plan(cfg, max_hops=None):
    """The bounded sample of the workload the CPU legs run: strided sources x >= 2(2M-1) hops
    (the delay line wraps), sized for ~1-2 s on a 16-core host."""
    hops = min(cfg.hops, max(2 * (2 * cfg.partitions - 1), 64)) if max_hops is None else min(max_hops, cfg.hops)
    per_lane_hop = cfg.partitions * (2 * cfg.hop + 1) * cfg.ears  # MAC complex products (cost proxy)
    lanes = int(max(1, min(cfg.sources, 64, 4.2e9 / (per_lane_hop * hops))))
    stride = max(1, cfg.sources // lanes)
    return list(range(0, stride * lanes, stride)), hops


def cpu_run(cfg, subset, n_hops, threads, want_output=True):
    """The reference's CPU path (oracle/_ref = the reference's own engine sources when built;
    else the restated oracle) over the sample: the bench's CPU baseline / reference arm and the
    checker of the GPU outputs — never the measured GPU path."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O

    kind = "reference" if O.ref_available() else "port"
    L = cfg.hop
    x = np.stack([W.white(cfg, s, 1, 0, n_hops * L, dtype=np.float64)[0] for s in subset])
    with O.using("ref" if kind == "reference" else "port"):
        if cfg.mode == "bank":
            bank = W.bank_irs(cfg, dtype=np.float64)
            sched = np.ascontiguousarray(W.schedule(cfg, 0, n_hops, 0, cfg.sources)[:, subset])
            secs, y = O.run_workload(L, cfg.partitions, len(subset), cfg.ears, n_hops, x, 1, bank_ir=bank,
                                     schedule=sched, threads=threads, want_output=want_output)
        else:
            n_sw = -(-n_hops // cfg.period)
            irs = np.stack([W.ir_items(cfg, [(s, e, k) for s in subset for e in range(cfg.ears)], dtype=np.float64)
                            .reshape(len(subset), cfg.ears, cfg.ir_length) for k in range(n_sw)])
            secs, y = O.run_workload(L, cfg.partitions, len(subset), cfg.ears, n_hops, x, 0, fresh_ir=irs,
                                     period=cfg.period, threads=threads, want_output=want_output)
    return secs, y, kind


def cpu_note(kind):
    if kind == "reference":
        return ("the reference's own proj/src/{spectral,partition,engine}.cpp compiled unmodified (-O3 -DNDEBUG, "
                "proj/CMakeLists.txt:8-10) against a minimal Eigen stand-in (oracle/_ref); lanes partitioned over "
                "std::threads (SPEC.md:221); timed region = process + partition like experiment.cpp:42-52")
    return ("fp64 C++ restatement of proj/src/{spectral,partition,engine}.cpp (oracle/, bit-identical to the "
            "reference on every config: tests/test_ref_pin.py); lanes over std::threads; timed region = process + "
            "partition like experiment.cpp:42-52")


def run_reference(args, cfg, rank):
    if rank != 0:  # the reference arm runs once, on rank 0
        return
    threads = W.host_threads()
    subset, n_hops = cpu_sample_plan(cfg, args.cpu_hops or None)
    vals, kind = [], "port"
    for i in range(args.warmup + args.steps):
        secs, _, kind = cpu_run(cfg, subset, n_hops, threads, want_output=False)
        if i >= args.warmup:
            vals.append(len(subset) * cfg.ears * n_hops * cfg.hop / secs)
    v = float(statistics.mean(vals))
    world = int(os.environ.get("WORLD_SIZE", 1))
    sample = (f"{len(subset)} sources (every {subset[1] - subset[0] if len(subset) > 1 else 1}th) x {cfg.ears} ear(s) "
              f"x {n_hops} hops of {cfg.name} per step (the same channels, hops, schedule / IRs and inputs as the "
              "GPU arm's workload)")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * len(subset) * cfg.ears * n_hops * cfg.hop / v,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, cfg.hops, 1, cfg.sources, "strong"),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": min(threads, len(subset)), "kind": kind,
                         "sample": sample, "note": cpu_note(kind)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "same_config": True,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- roofline
def fp32_peak_tflops(sms, mhz):
    return sms * 128 * 2 * mhz * 1e6 / 1e12


def roofline_block(cfg, summ_path, kern_ms, kern_n, hops_per_launch, distinct, clk, sms, pk, wide):
    """Measured sides of the dominant kernel's roofline, per launch, over the live launch time."""
    hbm = pk.get("hbm_gbs") or 6650.0
    l2pk = pk.get("l2_read_gbs")
    avg_ms = kern_ms / kern_n if kern_n else float("nan")
    t = avg_ms / 1e3
    sides, ncu = {}, None
    if summ_path.exists():
        sj = json.loads(summ_path.read_text())
        ph = sj.get("per_hop", {})
        ncu = {k: sj.get(k) for k in ("kernel", "source", "hops_per_launch", "duration_us_cold", "per_hop",
                                      "lts_throughput_pct", "dram_throughput_pct", "l2_hit_pct", "top_stalls")}
        ncu["file"] = f"profiles/{summ_path.name}"
        if ph.get("dram_bytes"):
            a = ph["dram_bytes"] * hops_per_launch / t / 1e9
            sides["hbm"] = {"achieved": a, "peak": hbm, "unit": "GB/s", "frac": a / hbm,
                            "bytes_per_hop": ph["dram_bytes"], "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        if ph.get("l2_read_bytes") and l2pk:
            a = (ph["l2_read_bytes"] + ph.get("l2_write_bytes", 0.0)) * hops_per_launch / t / 1e9
            sides["l2"] = {"achieved": a, "peak": l2pk, "unit": "GB/s", "frac": a / l2pk,
                           "bytes_per_hop": ph["l2_read_bytes"] + ph.get("l2_write_bytes", 0.0),
                           "peak_source": "profiles/l2_peak.json (scripts/l2_bw.cu, L2-resident reads, this pool)"}
    flops = W.flops_per_hop(cfg) * hops_per_launch
    mhz = (clk or {}).get("sm_mhz") or pk.get("sm_max_mhz") or 1965.0
    fpk = fp32_peak_tflops(sms, mhz)
    sides["fp32"] = {"achieved": flops / t / 1e12, "peak": fpk, "unit": "TFLOP/s", "frac": flops / t / 1e12 / fpk,
                     "flops_per_hop": W.flops_per_hop(cfg),
                     "flops_model": "cost.cpp:34-38 (MAC 8 B M per lane + the hop's forward / inverse transforms) "
                                    "+ for fresh-IR configs the K4 transforms of the switches (M per lane / period)",
                     "peak_source": f"{sms} SMs x 128 FP32 lanes x 2 x {mhz:.0f} MHz (median SM clock under load)"}
    bound = max(sides, key=lambda k: sides[k]["frac"])
    b = sides[bound]
    alg = W.bytes_per_hop(cfg, distinct_filters=distinct)
    k4 = None
    if cfg.mode == "fresh":  # the IR-switch path's bytes, reported beside the MAC's
        B = 2 * cfg.hop + 1
        k4 = {"bytes_per_hop": cfg.lanes * cfg.partitions * (2 * cfg.hop * 4 + 8 * B) / cfg.period,
              "note": "lanes x M x (2L taps x 4 B + B bins x 8 B) / period: IR slices read + partition spectra "
                      "written once per switch (the period tiles keep the spectra on chip, so only the taps move)"}
    return {
        "bound": bound, "achieved": b["achieved"], "peak": b["peak"], "unit": b["unit"], "frac": b["frac"],
        "switch_k4": k4,
        "traffic": (sides["hbm"]["bytes_per_hop"] * hops_per_launch) if "hbm" in sides else None,
        "sides": sides,
        "kernel": wide,
        "avg_launch_ms": avg_ms, "launches": kern_n, "hops_per_launch": hops_per_launch,
        "algorithmic": {"bytes_per_hop_8d": alg, "gbs": alg * hops_per_launch / t / 1e9,
                        "distinct_filters_per_hop": distinct,
                        "note": "SURVEY 8(d) compulsory bytes (every output re-reads M delay-line and M filter "
                                "spectra) over the launch time; the kernels reuse spectra across hops and channels "
                                "on chip / in L2, so this exceeds any single memory level's bandwidth"},
        "ncu": ncu,
        "timing": "avg launch time from a separate event-instrumented pass (events on the engine stream)",
    }


# ----------------------------------------------------------------------------- launcher
def spawn(args):
    """--gpus N without torchrun: re-launch this script under torch.distributed.run, one rank per GPU."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    log("spawning:", " ".join(cmd))
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"))
    return subprocess.call(cmd, env=env)


# ----------------------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--hops", type=int, default=0, help="override hops per step (default: the config's full length)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-hops", type=int, default=0, help="CPU sample hops (default >= 2(2M-1))")
    ap.add_argument("--latency-hops", type=int, default=300,
                    help="single-hop process() calls timed for the p50/p99 per-hop latency (0: skip)")
    ap.add_argument("--mix", default="p2p", choices=["p2p", "nccl"],
                    help="C3 cross-GPU mix: fused peer-memory kernels (default) or NCCL all-reduce")
    ap.add_argument("--one-gpu", action="store_true",
                    help="test harness: every rank on cuda:0 over gloo (the launcher, sharding and mix logic on one GPU)")
    ap.add_argument("--dump", default="", help="test harness: save each rank's outputs (and mix) as .npy here")
    ap.add_argument("--tune", action="append", default=[], metavar="KEY=VALUE",
                    help="engine tuning knob for an A/B run (tvolap_set_default_tuning; DESIGN.md §10)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    cfg = W.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg, rank)

    import torch

    from paper_2310_00319_b200 import _build, shard
    from paper_2310_00319_b200 import tvolap as T
    from paper_2310_00319_b200.tvolap import TvolapBankEngine, TvolapEngine, partition

    _build.build()
    for kv in args.tune:
        k, v = kv.split("=")
        T.set_default_tuning(k, int(v))
    if args.one_gpu:  # test harness: every rank on cuda:0, gloo (NCCL needs a GPU per rank)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev  # device of the tensors the process group reduces
    if world > 1:
        import torch.distributed as dist

        if args.one_gpu:
            dist.init_process_group("gloo")
            cdev = torch.device("cpu")
        else:
            dist.init_process_group("nccl", device_id=dev)
    L, M = cfg.hop, cfg.partitions
    H = args.hops or cfg.hops
    n_sw = -(-H // cfg.period)
    if args.scaling == "weak":
        lane0, S = shard.weak_lanes(cfg.sources, rank)
    else:
        lane0, S = shard.strong_lanes(cfg.sources, rank, world)
    lanes = S * cfg.ears
    lib = T.lib()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    # ---- inputs resident in HBM (device twins of the seeded generators), this rank's channels
    t0 = time.time()
    x = torch.empty((S, H * L), dtype=torch.float32, device=dev)
    T._check(lib.tvolap_gen_white_device(local, cfg.seed, lane0, S, 0, H * L, ctypes.c_void_p(x.data_ptr()), H * L))
    out = torch.empty((lanes, H * L), dtype=torch.float32, device=dev)

    def gen_irs(items, dst, arrays=None):
        if arrays is None:
            la = np.array([i[0] for i in items], np.int64)
            ea = np.array([i[1] for i in items], np.int64)
            ka = np.array([i[2] for i in items], np.int64)
            ta = np.array([W.t60_of(cfg, int(l), int(k)) for l, _, k in items], np.float64)
        else:
            la, ea, ka, ta = arrays
        T._check(lib.tvolap_gen_irs_device(local, cfg.seed, len(la), la.ctypes.data, ea.ctypes.data,
                                           ka.ctypes.data, ta.ctypes.data, W.FS, cfg.ir_length,
                                           ctypes.c_void_p(dst.data_ptr())))

    def fit_block(e):
        """Blocks never span a filter switch: cap the hop block at the period (C4: 8)."""
        j, _, _ = e.block_config()
        if cfg.period < j:
            e.set_block_config(max(2, 1 << (cfg.period.bit_length() - 1)))

    sched = mix = irs = None
    stream = torch.cuda.Stream(device=dev)
    chunk = n_sw
    if cfg.mode == "fresh":
        # a fresh seeded IR per (channel, switch), generated on the device. C4's 704 switches x 256
        # channels x 262144 taps (180 GB) do not fit: the step runs in chunks of periods whose sets
        # (<= 16 GB) are generated between the chunks' process_switching calls, outside the timed
        # intervals (the reference times process + partition, experiment.cpp:42-52)
        set_bytes = S * cfg.ir_length * 4
        chunk = int(max(1, min(n_sw, 16e9 // set_bytes)))
        irs = torch.empty((chunk, S, cfg.ir_length), dtype=torch.float32, device=dev)
        items = [(lane0 + s, 0, k) for k in range(n_sw) for s in range(S)]
        ir_arrays = (np.array([i[0] for i in items], np.int64), np.array([i[1] for i in items], np.int64),
                     np.array([i[2] for i in items], np.int64),
                     np.array([W.t60_of(cfg, int(l), int(k)) for l, _, k in items], np.float64))

        def gen_chunk(c0):
            stream.synchronize()  # the previous chunk's calls are done reading the sets
            c1 = min(n_sw, c0 + chunk)
            gen_irs(None, irs, tuple(a[c0 * S: c1 * S] for a in ir_arrays))

        if chunk >= n_sw:
            gen_chunk(0)
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
    log(f"[rank {rank}] {cfg.name}: channels {lane0}..{lane0 + S - 1}, generated {x.numel() * 4 / 1e6:.0f} MB input"
        f"{'' if irs is None else f' + {irs.numel() * 4 / 1e9:.2f} GB IRs'} in {time.time() - t0:.1f} s")
    eng.set_stream(stream.cuda_stream)
    comm = grp = None
    mix_path = None
    if mix is not None and world > 1:
        # C3: the fused peer-memory mix (one kernel per rank stores its partial into every rank's
        # gather buffer over NVLink, rank-ordered sums); NCCL through the C-ABI if IPC is unavailable
        if args.mix == "p2p":
            try:
                grp = shard.MixGroup(local, cfg.ears, H * L)
            except Exception as ex:  # noqa: BLE001
                log(f"[rank {rank}] peer-memory mix unavailable ({ex}); using NCCL")
            ok = torch.tensor([1 if grp is not None else 0], device=cdev)
            torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)  # every rank takes the same path
            if ok.item() == 1:
                mix_path = ("peer memory: tvolap_mix_scatter (per-GPU source sum + P2P stores into every rank's "
                            "gather slot) + rank-ordered tvolap_mix_gather")
            elif grp is not None:
                grp.close()
                grp = None
        if grp is None:
            comm = NcclComm(lib, rank, world, local)
            mix_path = "per-GPU mix kernel + ncclAllReduce (tvolap_mix_allreduce)"

    class ChunkTimer:
        """Sum of CUDA-event intervals (engine stream) around the chunks' process_switching calls."""

        def __init__(self):
            self.pairs = []

        def begin(self):
            self.pairs.append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
            self.pairs[-1][0].record(stream)

        def end(self):
            self.pairs[-1][1].record(stream)

        def total(self):
            return sum(a.elapsed_time(b) for a, b in self.pairs)

    def step(e, xs, outs, ir_set, sch, mx=None, timer=None):
        e.reset()
        if cfg.mode == "fresh" and ir_set is not None and ir_set.is_cuda:
            # the drive() loop (exchange before every period's hops), one call per chunk of periods
            for c0 in range(0, n_sw, chunk):
                c1 = min(n_sw, c0 + chunk)
                if chunk < n_sw:
                    gen_chunk(c0)  # this chunk's fresh IRs, outside the timed interval
                h0, h1 = c0 * cfg.period, min(H, c1 * cfg.period)
                if timer:
                    timer.begin()
                e.process_switching(xs[:, h0 * L: h1 * L], [ir_set[k - c0] for k in range(c0, c1)], cfg.period,
                                    out=outs[:, h0 * L: h1 * L])
                if timer:
                    timer.end()
        elif cfg.mode == "fresh":
            # e2e: host-pinned sets, every switch uploads a whole set (cycled when they do not all fit)
            e.process_switching(xs, [ir_set[k % ir_set.shape[0]] for k in range(n_sw)], cfg.period, out=outs)
        else:
            e.process_hops(xs, out=outs, schedule=sch)
            if mx is not None and outs.is_cuda and grp is not None:
                grp.allreduce(outs, S, H * L, mx, stream.cuda_stream)
            elif mx is not None and outs.is_cuda:
                T._check(lib.tvolap_mix_allreduce(local, S, cfg.ears, H * L, ctypes.c_void_p(outs.data_ptr()), H * L,
                                                  ctypes.c_void_p(mx.data_ptr()), H * L,
                                                  ctypes.c_void_p(comm.handle if comm else None),
                                                  ctypes.c_void_p(stream.cuda_stream)))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(local)
    tw0 = time.time()
    for _ in range(max(args.warmup, 3)):  # never fewer than 3 untimed steps before the timed region
        step(eng, x, out, irs, sched, mix)
    barrier()
    # steps far shorter than nvidia-smi's 20 ms sampling (C1: 0.1 ms): keep warming up on the same
    # work until the sampler has seen the GPU busy (the clocks line then covers warm-up + timed region)
    fill = 0
    while time.time() - tw0 < 0.5 and fill < 20000:
        for _ in range(16):
            step(eng, x, out, irs, sched, mix)
        fill += 16
        torch.cuda.synchronize()
    barrier()
    launches0 = eng.kernel_launches()
    wide0 = eng.wide_passes()
    chunked = cfg.mode == "fresh" and chunk < n_sw
    timer = ChunkTimer() if chunked else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start = time.time()
    ev0.record(stream)
    for _ in range(args.steps):
        step(eng, x, out, irs, sched, mix, timer)
    ev1.record(stream)
    barrier()
    t_end = time.time()
    clk = clocks.stop(t_start, t_end)
    elapsed = timer.total() if timer else ev0.elapsed_time(ev1)
    gpu_launches = eng.kernel_launches() - launches0 + (args.steps if mix is not None else 0)
    passes = eng.wide_passes() - wide0
    if args.dump:  # test harness: this rank's outputs of the timed steps (and the mix)
        os.makedirs(args.dump, exist_ok=True)
        np.save(os.path.join(args.dump, f"out_{rank}.npy"), out.cpu().numpy())
        if mix is not None:
            np.save(os.path.join(args.dump, f"mix_{rank}.npy"), mix.cpu().numpy())
        with open(os.path.join(args.dump, f"shard_{rank}.json"), "w") as f:
            json.dump({"lane0": lane0, "sources": S, "hops": H, "mix_path": mix_path}, f)
    # Per-launch kernel durations: a separate pass of the same steps with CUDA events around the
    # dominant launch on the engine stream (kept out of the timed region above).
    prof_steps = max(1, min(args.steps, 2))
    eng.set_profiling(True)
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ptimer = ChunkTimer() if chunked else None
    ev2.record(stream)
    for _ in range(prof_steps):
        step(eng, x, out, irs, sched, mix, ptimer)
    ev3.record(stream)
    barrier()
    kern_ms, kern_n = eng.kernel_time()
    eng.set_profiling(False)
    prof_elapsed = ptimer.total() if ptimer else ev2.elapsed_time(ev3)
    elapsed = shard.max_over_ranks(elapsed, cdev)
    ms_per_step = elapsed / args.steps
    total_sources = cfg.sources * (world if args.scaling == "weak" else 1)
    samples_per_step = total_sources * cfg.ears * H * L
    value = samples_per_step / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel
    pk = peaks()
    hops_per_launch = H * prof_steps / kern_n if kern_n else H
    if cfg.mode == "bank" and cfg.period == 1 and passes:
        kname = ("bank_mac_kernel (bank pass K3: one CTA per (hop tile, channel x 32-column chunk, partition group), "
                 f"{hops_per_launch:.0f} hops x {S} sources per launch; K1 / K5 / head / fix-up are separate launches)")
    elif passes:
        kname = (f"wide_mac_kernel (time-parallel pass: K4 of the tile's set + K3 + K5 + OLA per (channel, tile)), "
                 f"{hops_per_launch:.0f} hops x {S} sources per launch")
    else:
        kname = f"tvolap_block_kernel (K1-K5 fused, hop-blocked), {hops_per_launch:.0f} hops x {S} sources per launch"
    roofline = roofline_block(cfg, ROOT / "profiles" / f"ncu_summary_{cfg.name}.json", kern_ms, kern_n,
                              hops_per_launch, distinct * (S / cfg.sources), clk, sms, pk, kname)
    roofline["kernel_share_of_step"] = kern_ms / prof_elapsed if prof_elapsed else None

    # ---- e2e through the public API with pinned host buffers (H2D inputs [+ IRs, schedule], D2H outputs)
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        oh = torch.empty(tuple(out.shape), dtype=torch.float32, pin_memory=True)
        h2d = xh.numel() * 4
        if cfg.mode == "fresh":
            # pinned host sets (<= 8 GB): the device's first chunk of fresh sets; every switch
            # uploads a whole set (C4: 704 uploads cycle through 31 sets)
            n_e2e = int(max(1, min(n_sw, 8e9 // (S * cfg.ir_length * 4), chunk)))
            if chunk < n_sw:
                gen_chunk(0)
            irh = torch.empty((n_e2e,) + tuple(irs.shape[1:]), dtype=torch.float32, pin_memory=True)
            irh.copy_(irs[:n_e2e])
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
        e2e_s = shard.max_over_ranks(e2e_s, cdev)
        same = bool(torch.equal(oh, out.cpu())) if (cfg.mode != "fresh" or n_e2e >= n_sw) else None
        e2e = {"value": samples_per_step / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(oh.numel() * 4), "ms_per_step": e2e_s * 1e3,
               "timing": "host wall clock around each full pass incl. final synchronize",
               "matches_device_path": same,
               "path": "tvolap_process_hops / process_switching with pinned host buffers: chunked H2D || kernels "
                       "|| D2H pipeline on three streams"}
        del irh, eng2

    # ---- p50/p99 per-hop latency of the streaming API (one process() call per hop)
    latency = None
    if args.latency_hops:
        lat_eng = (TvolapBankEngine(bank, L, S, min_partitions=M, device=local) if cfg.mode == "bank"
                   else TvolapEngine(partition(ir0.T, L, M), device=local))
        lat_eng.set_stream(stream.cuda_stream)
        xin = torch.empty((S, L), dtype=torch.float32, pin_memory=True)
        yout = torch.empty((lanes, L), dtype=torch.float32, pin_memory=True)
        nl = min(args.latency_hops + 8, H)
        xsrc = x[:, : nl * L].cpu()
        sch_np = sched.cpu().numpy() if sched is not None else None
        gpu_ms, host_ms = [], []
        lat_eng.set_profiling(True)  # events around the one-hop kernel launches (engine stream)
        for h in range(nl):
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
        kms, kn = lat_eng.kernel_time()
        lat_eng.set_profiling(False)
        q = lambda v, p: float(np.percentile(v, p))  # noqa: E731
        # roofline of the streaming kernel: it reads every channel's M delay-line spectra and M filter
        # rows each hop (no reuse across hops), HBM-bound; ncu's DRAM bytes per launch over ncu's
        # (cold) duration, against MEASURED_PEAKS hbm_gbs (profiles/ncu_summary_<cfg>_hop.json)
        hop_rf = None
        hs = ROOT / "profiles" / f"ncu_summary_{cfg.name}_hop.json"
        if hs.exists():
            hj = json.loads(hs.read_text())
            ph = hj.get("per_hop", {})
            if ph.get("dram_bytes") and ph.get("duration_us"):
                hbm = peaks().get("hbm_gbs") or 6650.0
                a = ph["dram_bytes"] / (ph["duration_us"] * 1e-6) / 1e9
                hop_rf = {"bound": "hbm", "achieved": a, "peak": hbm, "unit": "GB/s", "frac": a / hbm,
                          "dram_bytes_per_hop": ph["dram_bytes"], "kernel_us_ncu_cold": ph["duration_us"],
                          "kernel_us_live": 1e3 * kms / kn if kn else None,
                          "kernel": hj.get("kernel"), "file": f"profiles/{hs.name}"}
        latency = {"hops": len(gpu_ms), "gpu_ms_p50": q(gpu_ms, 50), "gpu_ms_p99": q(gpu_ms, 99),
                   "kernel_roofline": hop_rf,
                   "host_ms_p50": q(host_ms, 50), "host_ms_p99": q(host_ms, 99),
                   "hop_period_ms": 1e3 * L / W.FS,
                   "streaming_value": S * cfg.ears * L / (statistics.median(host_ms) / 1e3),
                   "what": "one tvolap_process() call per hop (the reference's process() API) on pinned host "
                           "buffers: the one-hop kernel reads the hop and writes the outputs through their device "
                           "mapping (PCIe traffic inside the kernel; tuning zero_copy = 0: H2D copy, kernel, D2H "
                           "copy); CUDA events on the engine stream (gpu) and host wall clock (host); "
                           "streaming_value = channel-samples/s at the median host time"}
        del lat_eng

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded white noise + decaying-noise IRs generated on device)",
        "config": config_block(cfg, H, world, S, args.scaling), "clocks": clk, "gpu_launches": int(gpu_launches),
        "roofline": roofline, "e2e": e2e, "latency": latency,
        "realtime_factor": (H * L / W.FS) / (ms_per_step / 1e3),
        "warmup_clock_fill_steps": fill,
        "mix_path": mix_path,
        "tuning": dict(kv.split("=") for kv in args.tune) or "defaults",
        "path": {"passes_per_step": passes / args.steps,
                 "kind": "bank pass" if (cfg.mode == "bank" and cfg.period == 1 and passes) else
                         ("time-parallel pass" if passes else "hop-blocked launches")},
    }
    if chunked:
        line["config"]["ir_sets"] = (f"a fresh seeded IR per (channel, switch): {n_sw} switches per step in chunks of "
                                     f"{chunk} periods whose sets are generated on the device between the chunks' "
                                     "process_switching calls")
        line["timing"] = ("sum of CUDA-event intervals (engine stream) around each chunk's process_switching call; "
                          "the IR generation between them is outside the timed region (experiment.cpp:42-52 times "
                          "process + partition)")
    if e2e and cfg.mode == "fresh" and e2e["matches_device_path"] is None:
        e2e["ir_sets"] = (f"{n_e2e} pinned host sets cycled over the {n_sw} switches (each switch uploads a whole "
                          "set); outputs not comparable to the device path's fresh sets")

    # ---- CPU baseline + in-line parity (rank 0, N=1 only): the reference on a bounded sample
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = W.host_threads()
        subset, ch = cpu_sample_plan(cfg, args.cpu_hops or None)
        ch = min(ch, H)
        secs, yref, kind = cpu_run(cfg, subset, ch, threads, want_output=True)
        rows = [s * cfg.ears + e for s in subset for e in range(cfg.ears)]
        y = out[rows, : ch * L].double().cpu().numpy()
        rel = float(np.abs(y - yref).max() / np.abs(yref).max())
        secs1, _, _ = cpu_run(cfg, subset[:1], min(ch, 256), 1, want_output=False)
        sample = (f"{len(subset)} sources (every {subset[1] - subset[0] if len(subset) > 1 else 1}th) x "
                  f"{cfg.ears} ear(s) x {ch} hops of {cfg.name}")
        line["cpu_baseline"] = {
            "value": len(subset) * cfg.ears * ch * L / secs, "unit": UNIT, "cores": min(threads, len(subset)),
            "kind": kind, "sample": sample, "note": cpu_note(kind),
            "single_thread_value": cfg.ears * min(ch, 256) * L / secs1,
        }
        line["parity"] = {"rel_err_vs_reference": rel, "tolerance": 1e-4, "ok": rel <= 1e-4, "sample": sample,
                          "checked": "the bench's own device-path outputs of the timed pass vs the CPU reference",
                          "e2e_bit_identical_to_device_path": e2e["matches_device_path"] if e2e else None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm:
        comm.close()
    if grp:
        grp.close()
    if world > 1:
        torch.distributed.destroy_process_group()


class NcclComm:
    """An NCCL communicator made through the C-ABI (tvolap_nccl_*): rank 0's unique id is shared
    through torch.distributed, so a C++ host does the same with its own transport."""

    def __init__(self, lib, rank, world, device):
        import torch
        import torch.distributed as dist

        buf = (ctypes.c_char * 128)()
        if rank == 0:
            from paper_2310_00319_b200 import tvolap as T

            T._check(lib.tvolap_nccl_unique_id(buf))
        t = torch.tensor(list(bytes(buf)), dtype=torch.uint8, device=f"cuda:{device}")
        dist.broadcast(t, 0)
        raw = bytes(t.cpu().tolist())
        h = ctypes.c_void_p()
        from paper_2310_00319_b200 import tvolap as T

        T._check(lib.tvolap_nccl_comm_init(ctypes.byref(h), device, world, rank, raw))
        self.lib, self.handle = lib, h.value

    def close(self):
        if self.handle:
            self.lib.tvolap_nccl_comm_destroy(ctypes.c_void_p(self.handle))
            self.handle = None


if __name__ == "__main__":
    main()
