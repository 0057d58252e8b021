"""BASELINE.json workload configs and their seeded generators.

The five configs of /root/repo/BASELINE.json, with the defaults SURVEY.md §8(d)
recommends where BASELINE leaves a choice open (recorded in DESIGN.md):
  * FFT length is 4L, partitions are 2L taps (proj/include/tvolap/partition.hpp:30);
  * IRs are Gaussian x exp(-6.91 n / (T60 fs)), unit energy, for every config;
  * C3's bank holds 256 two-ear entries, input 10 s; C4 switches to fresh IRs.
Values come from libtvolap_workload.so (host) or the device twin in
libtvolap_b200.so — the same 64-bit words either way (csrc/workload.h).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

import numpy as np

FS = 48000.0
_WLIB = Path(__file__).resolve().parent / "lib" / "libtvolap_workload.so"
_wl = None


def wlib() -> C.CDLL:
    global _wl
    if _wl is None:
        L = C.CDLL(str(_WLIB))
        lg, u64, dp, vp = C.c_long, C.c_uint64, C.c_double, C.c_void_p
        L.tv_gen_white.argtypes = [u64, lg, lg, lg, lg, vp, vp, lg, C.c_int]
        L.tv_gen_white.restype = None
        L.tv_gen_irs.argtypes = [u64, lg, vp, vp, vp, vp, dp, lg, vp, vp, C.c_int]
        L.tv_gen_irs.restype = None
        L.tv_t60_c.argtypes = [u64, lg, lg, dp, dp]
        L.tv_t60_c.restype = dp
        L.tv_gen_schedule.argtypes = [u64, lg, lg, lg, C.c_int, vp, C.c_int]
        L.tv_gen_schedule.restype = None
        L.tv_rand64_c.argtypes = [u64, u64, u64]
        L.tv_rand64_c.restype = u64
        L.tv_gen_pink.argtypes = [u64, lg, vp]
        L.tv_gen_pink.restype = None
        L.tv_synthetic_binaural_ir.argtypes = [dp, lg, dp, u64, vp]
        L.tv_synthetic_binaural_ir.restype = C.c_int
        _wl = L
    return _wl


def host_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


@dataclass(frozen=True)
class Config:
    name: str
    hop: int                 # L
    partitions: int          # M (IR length = 2 L M)
    sources: int             # input lanes
    ears: int                # outputs per source
    seconds: float
    mode: str                # "fresh": new IR per lane every `period` hops; "bank": per-hop choice
    period: int              # hops between switches (fresh) / between re-draws (bank)
    n_bank: int = 0
    t60: tuple = (0.5, 0.5)  # T60 range in seconds
    mix: bool = False        # sum all source outputs into an `ears`-channel mix
    seed: int = 2310_00319

    @property
    def ir_length(self) -> int:
        return 2 * self.hop * self.partitions

    @property
    def lanes(self) -> int:
        return self.sources * self.ears

    @property
    def hops(self) -> int:
        return int(self.seconds * FS) // self.hop

    def scaled(self, **kw) -> "Config":
        d = dict(self.__dict__)
        d.update(kw)
        return Config(**d)


CONFIGS = {
    # C1: single channel, L=128, M=32, 10 s, two IRs alternating every 64 blocks.
    "C1": Config("C1", 128, 32, 1, 1, 10.0, "bank", 64, n_bank=2, t60=(0.5, 0.5)),
    # C2: 64 channels, L=256, M=64, own IR per channel, fresh IR every 16 blocks, 30 s.
    "C2": Config("C2", 256, 64, 64, 1, 30.0, "fresh", 16, t60=(0.3, 1.5)),
    # C3: 1024 sources x 2 ears, L=128, M=128, bank of 256 pairs, per-block choice, stereo mix.
    "C3": Config("C3", 128, 128, 1024, 2, 10.0, "bank", 1, n_bank=256, t60=(0.8, 0.8), mix=True),
    # C4: 256 channels, L=512, M=256, fresh IR every 8 blocks, 60 s.
    "C4": Config("C4", 512, 256, 256, 1, 60.0, "fresh", 8, t60=(4.0, 4.0)),
    # C5: 4096 channels, L=32, M=512, bank of 1024, per-block choice, 10 s.
    "C5": Config("C5", 32, 512, 4096, 1, 10.0, "bank", 1, n_bank=1024, t60=(0.4, 0.4)),
}


# ---------------------------------------------------------------- host generators
def white(cfg: Config, lane0: int, lanes: int, t0: int, n: int, dtype=np.float32,
          threads: Optional[int] = None) -> np.ndarray:
    """(lanes, n) uniform [-1,1) noise; float64 output holds the fp32-rounded values."""
    out = np.empty((lanes, n), dtype=dtype)
    p32 = out.ctypes.data if dtype == np.float32 else None
    p64 = out.ctypes.data if dtype == np.float64 else None
    wlib().tv_gen_white(cfg.seed, lane0, lanes, t0, n, p32, p64, n, threads or host_threads())
    return out


def t60_of(cfg: Config, lane: int, k: int) -> float:
    lo, hi = cfg.t60
    return wlib().tv_t60_c(cfg.seed, lane, k, lo, hi)


def ir_items(cfg: Config, items, dtype=np.float32, threads: Optional[int] = None) -> np.ndarray:
    """IRs for a list of (lane, ear, k) -> (len(items), ir_length)."""
    items = list(items)
    lanes = np.array([i[0] for i in items], dtype=np.int64)
    ears = np.array([i[1] for i in items], dtype=np.int64)
    ks = np.array([i[2] for i in items], dtype=np.int64)
    t60 = np.array([t60_of(cfg, int(l), int(k)) for l, _, k in items], dtype=np.float64)
    out = np.empty((len(items), cfg.ir_length), dtype=dtype)
    p32 = out.ctypes.data if dtype == np.float32 else None
    p64 = out.ctypes.data if dtype == np.float64 else None
    wlib().tv_gen_irs(cfg.seed, len(items), lanes.ctypes.data, ears.ctypes.data, ks.ctypes.data,
                      t60.ctypes.data, FS, cfg.ir_length, p32, p64, threads or host_threads())
    return out


def fresh_irs(cfg: Config, k: int, lane0: int = 0, lanes: Optional[int] = None, dtype=np.float32) -> np.ndarray:
    """IR set k (switch index) of the fresh-IR configs: (lanes, ears, ir_length)."""
    lanes = cfg.sources if lanes is None else lanes
    items = [(lane0 + s, e, k) for s in range(lanes) for e in range(cfg.ears)]
    return ir_items(cfg, items, dtype).reshape(lanes, cfg.ears, cfg.ir_length)


def bank_irs(cfg: Config, dtype=np.float32) -> np.ndarray:
    """Bank entries (n_bank, ears, ir_length); entry b is IR (lane=b, ear, k=0) of the bank stream."""
    items = [(b, e, 0) for b in range(cfg.n_bank) for e in range(cfg.ears)]
    return ir_items(cfg, items, dtype).reshape(cfg.n_bank, cfg.ears, cfg.ir_length)


def schedule(cfg: Config, hop0: int, n_hops: int, lane0: int = 0, lanes: Optional[int] = None) -> np.ndarray:
    """Bank choice per (hop, source): (n_hops, lanes) int32.

    C1 alternates its two IRs every `period` hops; C3/C5 draw uniformly every hop.
    """
    lanes = cfg.sources if lanes is None else lanes
    if cfg.name == "C1" or (cfg.n_bank == 2 and cfg.period > 1):
        h = np.arange(hop0, hop0 + n_hops)
        return np.repeat(((h // cfg.period) % 2).astype(np.int32)[:, None], lanes, axis=1)
    full = np.empty((n_hops, lane0 + lanes), dtype=np.int32)
    wlib().tv_gen_schedule(cfg.seed, hop0, n_hops, lane0 + lanes, cfg.n_bank, full.ctypes.data, host_threads())
    return np.ascontiguousarray(full[:, lane0:])


# ---------------------------------------------------------------- algorithmic bytes
def bytes_per_hop(cfg: Config, distinct_filters: Optional[float] = None, mix_outputs: Optional[int] = None) -> float:
    """Compulsory fp32 bytes per hop, B = 2L+1 bins.

    ring reads 8 B M S + filter reads 8 B M E F + ring write 8 B S + input 4 L S
    + output 4 L O + OLA state 48 L lanes.
    """
    L, M, S, E = cfg.hop, cfg.partitions, cfg.sources, cfg.ears
    B = 2 * L + 1
    F = cfg.sources if distinct_filters is None else distinct_filters
    O = cfg.lanes if mix_outputs is None else mix_outputs
    return 8 * B * M * S + 8 * B * M * E * F + 8 * B * S + 4 * L * S + 4 * L * O + 48 * L * cfg.lanes


def flops_per_hop(cfg: Config, with_switches: bool = True) -> float:
    """MAC + forward/inverse FFT flops per hop (reference cost model, cost.cpp:34-38), plus — for
    the fresh-IR configs — the filter partition transforms of the switches (partition.cpp:20-51:
    M transforms of the same size per lane and switch, spread over the period)."""
    L, M = cfg.hop, cfg.partitions
    B = 2 * L + 1
    fft = (5 * np.log2(2 * L) + 14) * 2 * L
    f = cfg.lanes * 8 * B * M + (cfg.sources + cfg.lanes) * fft
    if with_switches and cfg.mode == "fresh":
        f += cfg.lanes * M * fft / cfg.period
    return f


def gen_pink(seed: int, n: int) -> np.ndarray:
    """gen_pink (proj/src/signal_gen.cpp:42-59): (n,) fp64, bit-exact with the reference."""
    if n < 1:
        raise ValueError("gen_pink: need at least one sample")
    out = np.empty(n)
    wlib().tv_gen_pink(seed, n, out.ctypes.data)
    return out


def synthetic_binaural_ir(azimuth_deg: float, n_ir: int, fs: float = FS, seed: int = 7) -> np.ndarray:
    """synthetic_binaural_ir (proj/src/signal_gen.cpp:73-107): (n_ir, 2) fp64."""
    out = np.empty((2, n_ir))
    if wlib().tv_synthetic_binaural_ir(azimuth_deg, n_ir, fs, seed, out.ctypes.data):
        raise ValueError("synthetic_binaural_ir: response too short or bad sample rate")
    return np.ascontiguousarray(out.T)

