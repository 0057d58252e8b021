"""Python mirror of the reference's TVOLAP operator interface, over the C-ABI.

Same names, argument meaning and error behaviour as the reference C++ API so the
parity tests read like the reference's own tests:

  hann_window(hop)                          proj/src/partition.cpp:10-18
  forward_real / inverse_real / mac         proj/src/spectral.cpp:99-172
  partition(ir, hop, min_partitions)        proj/src/partition.cpp:20-51
  TvolapEngine(set)                         proj/include/tvolap/engine.hpp:33-94
  TvolapProcessor(ir, hop), make_processor  proj/include/tvolap/reference.hpp:202-226

Every call goes through libtvolap_b200.so (include/tvolap_b200.h); there is no
CPU fallback — importing works anywhere, but an engine needs a B200. Exceptions
mirror proj/include/tvolap/errors.hpp. Sample arrays follow the reference's
Eigen layout: `process` takes and returns (L rows x C cols) arrays; multi-hop
calls take (lanes, samples) arrays or torch tensors (device tensors stay on the
device, the call is then asynchronous on the engine stream).
"""
from __future__ import annotations

import ctypes as C
from contextlib import contextmanager
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np

# TVOLAP_LIB: a diagnostic build (scripts/, _build.build_variant) instead of the in-tree library
_LIB_PATH = Path(os.environ.get("TVOLAP_LIB") or Path(__file__).resolve().parent / "lib" / "libtvolap_b200.so")


# ---------------------------------------------------------------- errors (errors.hpp)
class InvalidSizeError(ValueError):
    """tvolap::InvalidSizeError (errors.hpp:10)."""


class InvalidInputError(ValueError):
    """tvolap::InvalidInputError (errors.hpp:16)."""


class InvalidSpectrumError(ValueError):
    """tvolap::InvalidSpectrumError (errors.hpp:28)."""


class IncompatibleFilterError(ValueError):
    """tvolap::IncompatibleFilterError (errors.hpp:34)."""


class InvalidConfigurationError(ValueError):
    """tvolap::InvalidConfigurationError (errors.hpp:40)."""


class CudaError(RuntimeError):
    """Device failure (no reference analogue): the engine never falls back to the CPU."""


class SwitchInProgressError(RuntimeError):
    """tvolap::SwitchInProgressError (errors.hpp:46) — a crossfade is already running."""


_ERRORS = {
    1: InvalidSizeError,
    2: InvalidInputError,
    3: InvalidConfigurationError,
    4: IncompatibleFilterError,
    5: InvalidSpectrumError,
    6: CudaError,
    7: SwitchInProgressError,
}

_lib = None


def lib() -> C.CDLL:
    """Load libtvolap_b200.so (raises if it was not built — no fallback path exists)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise CudaError(f"{_LIB_PATH} is missing; run __graft_entry__.build()")
        L = C.CDLL(str(_LIB_PATH))
        vp, lg, ip, fp = C.c_void_p, C.c_long, C.c_int, C.c_void_p
        sig = {
            "tvolap_last_error": (C.c_char_p, []),
            "tvolap_version": (C.c_char_p, []),
            "tvolap_create": (ip, [C.POINTER(vp), ip, lg, lg, lg, fp, lg]),
            "tvolap_create_bank": (ip, [C.POINTER(vp), ip, lg, lg, lg, lg, lg, fp, lg]),
            "tvolap_destroy": (ip, [vp]),
            "tvolap_process": (ip, [vp, fp, lg, lg, lg, fp, lg]),
            "tvolap_process_hops": (ip, [vp, fp, lg, fp, lg, lg, fp]),
            "tvolap_process_switching": (ip, [vp, fp, lg, fp, lg, lg, lg, vp, lg]),
            "tvolap_exchange_filter": (ip, [vp, fp, lg, lg]),
            "tvolap_select_bank": (ip, [vp, fp]),
            "tvolap_reset": (ip, [vp]),
            "tvolap_hop": (lg, [vp]),
            "tvolap_channels": (lg, [vp]),
            "tvolap_output_channels": (lg, [vp]),
            "tvolap_partition_count": (lg, [vp]),
            "tvolap_delay_line_depth": (lg, [vp]),
            "tvolap_latency": (lg, [vp]),
            "tvolap_switching_latency": (lg, [vp]),
            "tvolap_stream_delay": (lg, [vp]),
            "tvolap_hops_processed": (lg, [vp]),
            "tvolap_op_counts": (ip, [vp, fp, fp, fp]),
            "tvolap_set_stream": (ip, [vp, vp]),
            "tvolap_synchronize": (ip, [vp]),
            "tvolap_set_host_async": (ip, [vp, ip]),
            "tvolap_set_profiling": (ip, [vp, ip]),
            "tvolap_kernel_time": (ip, [vp, fp, fp]),
            "tvolap_launch_config": (ip, [vp, fp, fp]),
            "tvolap_set_launch_config": (ip, [vp, ip, ip]),
            "tvolap_kernel_launches": (C.c_uint64, [vp]),
            "tvolap_wide_passes": (C.c_uint64, [vp]),
            "tvolap_ring_launches": (C.c_uint64, [vp]),
            "tvolap_set_block_config": (ip, [vp, ip, lg]),
            "tvolap_set_tuning": (ip, [vp, C.c_char_p, lg]),
            "tvolap_set_create": (ip, [C.POINTER(vp), ip, lg, lg, lg, fp, lg]),
            "tvolap_set_release": (ip, [vp]),
            "tvolap_set_geometry": (ip, [vp, fp, fp, fp, fp]),
            "tvolap_set_spectra": (ip, [vp, fp]),
            "tvolap_set_reassemble": (ip, [vp, fp]),
            "tvolap_create_from_set": (ip, [C.POINTER(vp), vp]),
            "tvolap_exchange_set": (ip, [vp, vp]),
            "tvolap_get_tuning": (ip, [vp, C.c_char_p, C.POINTER(lg)]),
            "tvolap_set_default_tuning": (ip, [C.c_char_p, lg]),
            "tvolap_reset_default_tuning": (ip, []),
            "tvolap_tuning_keys": (C.c_char_p, []),
            "tvolap_block_config": (ip, [vp, fp, fp, fp]),
            "tvolap_forward_real": (ip, [ip, lg, lg, fp, fp]),
            "tvolap_inverse_real": (ip, [ip, lg, lg, fp, fp]),
            "tvolap_mac": (ip, [ip, lg, lg, fp, fp, fp, fp]),
            "tvolap_hann_window": (ip, [lg, fp]),
            "tvolap_partition": (ip, [ip, lg, lg, lg, fp, lg, fp, fp]),
            "tvolap_gen_white_device": (ip, [ip, C.c_uint64, lg, lg, lg, lg, fp, lg]),
            "tvolap_gen_irs_device": (ip, [ip, C.c_uint64, lg, fp, fp, fp, fp, C.c_double, lg, fp]),
            "tvolap_mix_device": (ip, [ip, lg, lg, lg, fp, lg, fp, lg, vp]),
            "tvolap_mix_allreduce": (ip, [ip, lg, lg, lg, fp, lg, fp, lg, vp, vp]),
            "tvolap_nccl_unique_id": (ip, [vp]),
            "tvolap_nccl_comm_init": (ip, [C.POINTER(vp), ip, ip, ip, vp]),
            "tvolap_nccl_comm_destroy": (ip, [vp]),
            "tvolap_mix_group_create": (ip, [C.POINTER(vp), ip, ip, ip, lg, lg, vp]),
            "tvolap_mix_group_open": (ip, [vp, vp]),
            "tvolap_mix_scatter": (ip, [vp, lg, lg, fp, lg, vp]),
            "tvolap_mix_gather": (ip, [vp, lg, fp, lg, vp]),
            "tvolap_mix_group_destroy": (ip, [vp]),
            "tvolap_cmp_create": (ip, [C.POINTER(vp), ip, ip, lg, lg, fp, lg, lg, lg, ip]),
            "tvolap_cmp_destroy": (ip, [vp]),
            "tvolap_cmp_process_hops": (ip, [vp, fp, lg, fp, lg, lg]),
            "tvolap_cmp_set_filter": (ip, [vp, fp, lg, lg, lg]),
            "tvolap_cmp_switch_filter": (ip, [vp, fp, lg, lg, lg, lg, ip]),
            "tvolap_cmp_reset": (ip, [vp]),
            "tvolap_cmp_geometry": (ip, [vp, fp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name, None)
            if f is None:  # an older diagnostic build (TVOLAP_LIB); tests check the real exports
                continue
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


EXPORTED_SYMBOLS = (
    "tvolap_last_error tvolap_version tvolap_create tvolap_create_bank tvolap_destroy tvolap_process "
    "tvolap_process_hops tvolap_process_switching tvolap_exchange_filter tvolap_select_bank tvolap_reset tvolap_hop tvolap_channels "
    "tvolap_output_channels tvolap_partition_count tvolap_delay_line_depth tvolap_latency "
    "tvolap_switching_latency tvolap_stream_delay tvolap_hops_processed tvolap_op_counts tvolap_set_stream "
    "tvolap_synchronize tvolap_set_host_async tvolap_set_profiling tvolap_kernel_time tvolap_launch_config tvolap_set_launch_config tvolap_kernel_launches tvolap_wide_passes tvolap_ring_launches tvolap_set_block_config tvolap_block_config "
    "tvolap_set_create tvolap_set_release tvolap_set_geometry tvolap_set_spectra tvolap_set_reassemble "
    "tvolap_create_from_set tvolap_exchange_set "
    "tvolap_set_tuning tvolap_get_tuning tvolap_set_default_tuning tvolap_reset_default_tuning tvolap_tuning_keys "
    "tvolap_forward_real tvolap_inverse_real tvolap_mac tvolap_hann_window tvolap_partition "
    "tvolap_gen_white_device tvolap_gen_irs_device tvolap_mix_device tvolap_mix_allreduce tvolap_nccl_unique_id "
    "tvolap_nccl_comm_init tvolap_nccl_comm_destroy "
    "tvolap_mix_group_create tvolap_mix_group_open tvolap_mix_scatter tvolap_mix_gather tvolap_mix_group_destroy "
    "tvolap_cmp_create tvolap_cmp_destroy tvolap_cmp_process_hops tvolap_cmp_set_filter tvolap_cmp_switch_filter "
    "tvolap_cmp_reset tvolap_cmp_geometry"
).split()


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().tvolap_last_error().decode()
        raise _ERRORS.get(rc, CudaError)(msg)


def _ptr(x):
    """(pointer, keepalive) for a float32/int32 numpy array or a torch tensor."""
    if x is None:
        return None, None
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr()), x
    return C.c_void_p(x.ctypes.data), x


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


# ---------------------------------------------------------------- spectral (spectral.hpp)
def is_power_of_two(n: int) -> bool:
    """spectral.hpp:31."""
    return n > 0 and (n & (n - 1)) == 0


def hann_window(hop: int) -> np.ndarray:
    """Periodic Hann of length 2L, peak 2 (partition.cpp:10-18)."""
    w = np.empty(2 * max(hop, 0), dtype=np.float32)
    _check(lib().tvolap_hann_window(hop, w.ctypes.data if w.size else None))
    return w


def forward_real(block, device: int = 0) -> np.ndarray:
    """Unscaled real FFT -> n/2+1 complex bins (spectral.cpp:99-125); batched over leading axes."""
    x = _f32(block)
    n = x.shape[-1] if x.ndim else 0
    batch = int(np.prod(x.shape[:-1])) if x.ndim > 1 else 1
    out = np.empty(x.shape[:-1] + (n // 2 + 1, 2), dtype=np.float32)
    _check(lib().tvolap_forward_real(device, n, batch, x.ctypes.data if x.size else None,
                                     out.ctypes.data if out.size else None))
    return out[..., 0] + 1j * out[..., 1]


def inverse_real(bins, n: Optional[int] = None, device: int = 0) -> np.ndarray:
    """Inverse of forward_real incl. 1/n (spectral.cpp:127-158)."""
    b = np.asarray(bins)
    nb = b.shape[-1]
    n = 2 * (nb - 1) if n is None else n
    if nb != n // 2 + 1:
        raise InvalidSizeError(f"inverse_real: expected {n // 2 + 1} bins, got {nb}")
    inter = _f32(np.stack([b.real, b.imag], axis=-1))
    batch = int(np.prod(b.shape[:-1])) if b.ndim > 1 else 1
    out = np.empty(b.shape[:-1] + (n,), dtype=np.float32)
    _check(lib().tvolap_inverse_real(device, n, batch, inter.ctypes.data, out.ctypes.data))
    return out


def mac(acc, a, b, device: int = 0) -> np.ndarray:
    """acc + a*b per bin (spectral.cpp:160-172)."""
    acc, a, b = (np.asarray(v) for v in (acc, a, b))
    if not (acc.shape == a.shape == b.shape):
        raise InvalidSizeError("mac: bin counts differ")
    st = [_f32(np.stack([v.real, v.imag], axis=-1)) for v in (acc, a, b)]
    out = np.empty_like(st[0])
    nb = acc.shape[-1]
    batch = acc.size // nb
    _check(lib().tvolap_mac(device, nb, batch, st[0].ctypes.data, st[1].ctypes.data, st[2].ctypes.data,
                            out.ctypes.data))
    return out[..., 0] + 1j * out[..., 1]


# ---------------------------------------------------------------- partition (partition.hpp)
@dataclass
class FilterPartitionSet:
    """partition.hpp:21-32: immutable, shared. Keeps the fp32 taps it was built from; the partition
    spectra live on the device (tvolap_set_create, one K4 per device on first use) and engines
    take / exchange to them in O(1) (tvolap_create_from_set / tvolap_exchange_set)."""

    hop: int
    partition_count: int
    channels: int
    source_length: int
    taps: np.ndarray = field(repr=False)  # (channels, source_length) fp32
    normalization_gain: float = 0.5
    sample_rate: float = 48000.0
    _dev: dict = field(default_factory=dict, repr=False, compare=False)  # device -> tvolap_set*

    def transform_length(self) -> int:
        return 4 * self.hop

    def padded_length(self) -> int:
        return 2 * self.hop * self.partition_count

    def device_set(self, device: int = 0):
        """The set's device-resident spectra on `device` (created once, then shared)."""
        h = self._dev.get(device)
        if h is None:
            h = C.c_void_p()
            _check(lib().tvolap_set_create(C.byref(h), device, self.hop, self.channels, self.source_length,
                                           self.taps.ctypes.data, self.partition_count))
            self._dev[device] = h
        return h

    def __del__(self):
        for h in getattr(self, "_dev", {}).values():
            if h and _lib is not None:
                _lib.tvolap_set_release(h)
        self._dev = {}

    def spectra(self, device: int = 0) -> np.ndarray:
        """(channels, M, 2L+1) complex partition spectra (the device set's)."""
        nb = 2 * self.hop + 1
        out = np.empty((self.channels, self.partition_count, nb, 2), dtype=np.float32)
        _check(lib().tvolap_set_spectra(self.device_set(device), out.ctypes.data))
        return out[..., 0] + 1j * out[..., 1]


def partition(ir, hop: int, min_partitions: int = 1, sample_rate: float = 48000.0) -> FilterPartitionSet:
    """partition(ir, hop, min_partitions) (partition.cpp:20-51). `ir`: (taps,) or (taps, channels) like Eigen."""
    h = np.asarray(ir, dtype=np.float64)
    if h.ndim == 1:
        h = h[:, None]
    if h.size == 0 or h.shape[0] < 1 or h.shape[1] < 1:
        raise InvalidInputError("partition: impulse response is empty")
    if hop < 2 or not is_power_of_two(4 * hop):
        raise InvalidSizeError(f"partition: 4L must be a power of two, got L = {hop}")
    slice_ = 2 * hop
    m = max(-(-h.shape[0] // slice_), max(min_partitions, 1))
    taps = np.ascontiguousarray(h.T, dtype=np.float32)
    return FilterPartitionSet(hop, m, h.shape[1], h.shape[0], taps, sample_rate=sample_rate)


def reassemble(s: FilterPartitionSet, device: int = 0) -> np.ndarray:
    """reassemble(set) (partition.hpp:43, partition.cpp:53-65) from the device spectra:
    (M * 2L, channels), the response zero-padded to M * 2L taps."""
    out = np.empty((s.channels, 2 * s.hop * s.partition_count), dtype=np.float32)
    _check(lib().tvolap_set_reassemble(s.device_set(device), out.ctypes.data))
    return np.ascontiguousarray(out.T)


# ---------------------------------------------------------------- engine (engine.hpp)
class TvolapEngine:
    """B200 TvolapEngine (engine.hpp:33-94) behind tvolap_create / tvolap_process."""

    def __init__(self, filter: FilterPartitionSet, device: int = 0):
        if filter is None:
            raise InvalidConfigurationError("engine requires a filter partition set")
        h = C.c_void_p()
        _check(lib().tvolap_create_from_set(C.byref(h), filter.device_set(device)))  # engine.hpp:35
        self._h = h
        self._filter = filter
        self.device = device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.tvolap_destroy(h)
            self._h = None

    # getters (engine.hpp:38-50)
    def hop(self) -> int:
        return lib().tvolap_hop(self._h)

    def channels(self) -> int:
        return lib().tvolap_channels(self._h)

    def partition_count(self) -> int:
        return lib().tvolap_partition_count(self._h)

    def delay_line_depth(self) -> int:
        return lib().tvolap_delay_line_depth(self._h)

    def latency(self) -> int:
        return lib().tvolap_latency(self._h)

    def switching_latency(self) -> int:
        return lib().tvolap_switching_latency(self._h)

    def stream_delay(self) -> int:
        return lib().tvolap_stream_delay(self._h)

    def filter(self) -> FilterPartitionSet:
        return self._filter

    def exchange_filter(self, next: Optional[FilterPartitionSet]) -> None:
        """engine.hpp:55, engine.cpp:37-48: validate, stage (O(1): the set's device spectra are read in
        place, no transform); latched at the next process(), last staged wins."""
        if next is None:
            raise IncompatibleFilterError("replacement filter is null")
        if next.hop != self.hop():
            raise IncompatibleFilterError("replacement filter hop differs")
        if next.partition_count != self.partition_count():
            raise IncompatibleFilterError("replacement filter partition count differs")
        if next.channels != self.channels():
            raise IncompatibleFilterError("replacement filter channel count differs")
        _check(lib().tvolap_exchange_set(self._h, next.device_set(self.device)))
        self._filter = next

    def exchange_ir(self, ir) -> None:
        """Stage a replacement IR given as (channels, taps) — numpy or a device tensor (no host copy)."""
        if ir.shape[0] != self.channels():
            raise IncompatibleFilterError("replacement filter channel count differs")
        if -(-ir.shape[1] // (2 * self.hop())) > self.partition_count():
            raise IncompatibleFilterError("replacement filter partition count differs")
        if not hasattr(ir, "data_ptr"):
            ir = _f32(ir)
        p, _k = _ptr(ir)
        _check(lib().tvolap_exchange_filter(self._h, p, ir.shape[1], ir.shape[0]))

    def process(self, input) -> np.ndarray:
        """One hop: (L, C) in -> (L, C) out (engine.cpp:60-106)."""
        x = np.asarray(input, dtype=np.float32)
        if x.ndim == 1:
            x = x[:, None]
        rows, cols = x.shape
        xf = np.ascontiguousarray(x.T)  # lane-major, like Eigen's column-major storage
        out = np.empty((self.channels_out(), max(rows, 1)), dtype=np.float32)
        _check(lib().tvolap_process(self._h, xf.ctypes.data, max(rows, 1), rows, cols, out.ctypes.data,
                                    max(rows, 1)))
        return out.T.copy()

    def channels_out(self) -> int:
        return lib().tvolap_output_channels(self._h)

    def process_hops(self, x, out=None, schedule=None):
        """n hops at once. x: (lanes, n*L) numpy array or torch tensor (host or device)."""
        L = self.hop()
        lanes, total = x.shape[0], x.shape[-1]
        if total % L:
            raise InvalidSizeError("process_hops: sample count is not a whole number of hops")
        n = total // L
        if out is None:
            if hasattr(x, "data_ptr"):
                import torch

                out = torch.empty((self.channels_out(), total), dtype=torch.float32, device=x.device)
            else:
                out = np.empty((self.channels_out(), total), dtype=np.float32)
        if not hasattr(x, "data_ptr"):
            x = _f32(x)
        _check_buffer(x, self.channels(), total, "process_hops input")
        _check_buffer(out, self.channels_out(), total, "process_hops output")
        if schedule is not None:
            if not hasattr(schedule, "data_ptr"):
                schedule = np.ascontiguousarray(schedule, np.int32)
            _check_buffer(schedule, n, self.channels(), "process_hops schedule", "int32")
            if n > 1 and _stride(schedule) != self.channels():
                raise InvalidInputError("process_hops schedule: rows must be dense (n_hops, sources)")
        xp, _k1 = _ptr(x)
        op, _k2 = _ptr(out)
        sp, _k3 = _ptr(schedule)
        _check(lib().tvolap_process_hops(self._h, xp, _stride(x), op, _stride(out), n, sp))
        return out

    def process_switching(self, x, irs, period: int, out=None):
        """n hops with a filter switch every `period` hops: the same as
        `for k: exchange_ir(irs[k]) (unless None); process_hops(period hops)`.
        irs: sequence of (lanes, taps) IR arrays / tensors (None = no switch at k), one per period.
        With device tensors everywhere this is one launch (tvolap_process_switching)."""
        L = self.hop()
        lanes, total = x.shape[0], x.shape[-1]
        if total % L:
            raise InvalidSizeError("process_switching: sample count is not a whole number of hops")
        n = total // L
        nsw = -(-n // period)
        if len(irs) < nsw:
            raise InvalidInputError(f"process_switching: {nsw} switch slots needed, got {len(irs)}")
        if out is None:
            if hasattr(x, "data_ptr"):
                import torch

                out = torch.empty((self.channels_out(), total), dtype=torch.float32, device=x.device)
            else:
                out = np.empty((self.channels_out(), total), dtype=np.float32)
        if not hasattr(x, "data_ptr"):
            x = _f32(x)
        _check_buffer(x, self.channels(), total, "process_switching input")
        _check_buffer(out, self.channels_out(), total, "process_switching output")
        keep, ptrs, taps = [], (C.c_void_p * nsw)(), 0
        for k in range(nsw):
            ir = irs[k]
            if ir is None:
                ptrs[k] = None
                continue
            if not hasattr(ir, "data_ptr"):
                ir = _f32(ir)
            if ir.shape[0] != self.channels():
                raise IncompatibleFilterError("replacement filter channel count differs")
            if taps and ir.shape[-1] != taps:
                raise InvalidInputError("process_switching: all IRs must have the same length")
            taps = ir.shape[-1]
            if _stride(ir) != taps:
                raise InvalidInputError("process_switching: IRs must be dense (lanes, taps)")
            p, k2 = _ptr(ir)
            keep.append(k2)
            ptrs[k] = p.value
        xp, _k1 = _ptr(x)
        op, _k2 = _ptr(out)
        _check(lib().tvolap_process_switching(self._h, xp, _stride(x), op, _stride(out), n, period,
                                              C.cast(ptrs, C.c_void_p), taps))
        return out

    def reset(self) -> None:
        _check(lib().tvolap_reset(self._h))

    def op_counts(self):
        """EngineOpCounts (engine.hpp:17-21): (forward_transforms, inverse_transforms, spectral_macs)."""
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().tvolap_op_counts(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return OpCounts(a.value, b.value, c.value)

    def hops_processed(self) -> int:
        return lib().tvolap_hops_processed(self._h)

    def set_stream(self, stream_handle: int) -> None:
        _check(lib().tvolap_set_stream(self._h, C.c_void_p(stream_handle)))

    def set_profiling(self, enable: bool = True) -> None:
        _check(lib().tvolap_set_profiling(self._h, int(enable)))

    def kernel_time(self):
        """(total device ms, launches) of the fused hop kernel since profiling was enabled."""
        ms, n = C.c_double(), C.c_long()
        _check(lib().tvolap_kernel_time(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def set_host_async(self, enable: bool = True) -> None:
        _check(lib().tvolap_set_host_async(self._h, int(enable)))

    def synchronize(self) -> None:
        _check(lib().tvolap_synchronize(self._h))

    def launch_config(self):
        p, t = C.c_int(), C.c_int()
        _check(lib().tvolap_launch_config(self._h, C.byref(p), C.byref(t)))
        return p.value, t.value

    def set_launch_config(self, ctas_per_source: int = 0, threads: int = 0) -> None:
        _check(lib().tvolap_set_launch_config(self._h, ctas_per_source, threads))

    def set_block_config(self, hops_per_block: int = 0, block_min: int = 0) -> None:
        _check(lib().tvolap_set_block_config(self._h, hops_per_block, block_min))

    def block_config(self):
        j, b, q = C.c_int(), C.c_long(), C.c_int()
        _check(lib().tvolap_block_config(self._h, C.byref(j), C.byref(b), C.byref(q)))
        return j.value, b.value, q.value

    def kernel_launches(self) -> int:
        return lib().tvolap_kernel_launches(self._h)

    def set_tuning(self, key: str, value: int) -> None:
        """A/B knob of this engine (tvolap_set_tuning; keys: tuning_keys())."""
        _check(lib().tvolap_set_tuning(self._h, key.encode(), int(value)))

    def get_tuning(self, key: str) -> int:
        v = C.c_long()
        _check(lib().tvolap_get_tuning(self._h, key.encode(), C.byref(v)))
        return v.value

    def wide_passes(self) -> int:
        """Time-parallel passes run (device-resident switching calls, csrc/tvolap_wide.cu)."""
        return lib().tvolap_wide_passes(self._h)

    def ring_launches(self) -> int:
        """One-hop launches that ran on the persistent bulk-copy ring kernel (bank engines)."""
        return lib().tvolap_ring_launches(self._h)


def tuning_keys():
    return lib().tvolap_tuning_keys().decode().split(",")


def set_default_tuning(key: str, value: int) -> None:
    """Value engines created afterwards start with (process-wide launch knobs take effect at once)."""
    _check(lib().tvolap_set_default_tuning(key.encode(), int(value)))


def reset_default_tuning() -> None:
    _check(lib().tvolap_reset_default_tuning())


@contextmanager
def default_tuning(**knobs):
    """with default_tuning(wide=0): ... — engines created inside start with these knobs."""
    for k, v in knobs.items():
        set_default_tuning(k, v)
    try:
        yield
    finally:
        reset_default_tuning()


@dataclass
class OpCounts:
    forward_transforms: int
    inverse_transforms: int
    spectral_macs: int


def _check_buffer(a, rows: int, total: int, what: str, dtype_name: str = "float32"):
    """Shape / dtype / layout of a caller buffer before its pointer crosses the C-ABI: a short or
    mistyped buffer would be read or written out of bounds there (engine.cpp:66-67 raises
    InvalidInputError on a channel mismatch)."""
    if a.ndim != 2 or a.shape[0] != rows or a.shape[-1] != total:
        raise InvalidInputError(f"{what}: expected shape ({rows}, {total}), got {tuple(a.shape)}")
    if hasattr(a, "data_ptr"):
        if str(a.dtype) != "torch." + dtype_name:
            raise InvalidInputError(f"{what}: expected torch.{dtype_name}, got {a.dtype}")
        if a.shape[-1] > 1 and a.stride(-1) != 1:
            raise InvalidInputError(f"{what}: the sample axis must be contiguous (unit stride)")
    else:
        if a.dtype != np.dtype(dtype_name):
            raise InvalidInputError(f"{what}: expected {dtype_name}, got {a.dtype}")
        if a.shape[-1] > 1 and a.strides[-1] != a.itemsize:
            raise InvalidInputError(f"{what}: the sample axis must be contiguous (unit stride)")
    if a.shape[0] > 1 and _stride(a) < total:
        raise InvalidInputError(f"{what}: lane stride shorter than the row")


def _stride(a) -> int:
    """Lane stride in elements (a size-1 leading dim may carry an arbitrary stride: use the row length)."""
    if a.shape[0] == 1:
        return a.shape[-1]
    if hasattr(a, "stride") and callable(a.stride):
        return a.stride(0)
    return a.strides[0] // a.itemsize


class TvolapBankEngine(TvolapEngine):
    """Bank engine (configs C1/C3/C5): sources x ears lanes over a pre-partitioned IR bank.

    bank_ir: (n_bank, ears, taps). Selection per source via select_bank() (staged,
    latched next hop) or a per-hop schedule in process_hops().
    """

    def __init__(self, bank_ir, hop: int, sources: int, min_partitions: int = 1, device: int = 0):
        b = bank_ir if hasattr(bank_ir, "data_ptr") else _f32(bank_ir)
        if b.ndim == 2:
            b = b[:, None, :]
        n_bank, ears, taps = b.shape
        h = C.c_void_p()
        bp, _keep = _ptr(b)
        _check(lib().tvolap_create_bank(C.byref(h), device, hop, sources, ears, n_bank, taps, bp, min_partitions))
        self._h = h
        self._filter = None
        self.device = device
        self.n_bank = n_bank
        self.ears = ears

    def select_bank(self, idx) -> None:
        i = np.ascontiguousarray(idx, dtype=np.int32)
        _check(lib().tvolap_select_bank(self._h, i.ctypes.data))

    def exchange_filter(self, next):  # bank engines switch by selection
        raise InvalidConfigurationError("exchange_filter on a bank engine; use select_bank")


# ---------------------------------------------------------------- processor facade (reference.hpp)
class TvolapProcessor:
    """TvolapProcessor(ir, hop) facade (reference.cpp:328-342)."""

    def __init__(self, ir, hop: int, device: int = 0):
        self._engine = TvolapEngine(partition(ir, hop), device=device)

    def name(self) -> str:
        return "tvolap"

    def hop(self) -> int:
        return self._engine.hop()

    def channels(self) -> int:
        return self._engine.channels()

    def latency(self) -> int:
        return self._engine.latency()

    def stream_delay(self) -> int:
        return self._engine.stream_delay()

    def switching_latency(self) -> int:
        return self._engine.switching_latency()

    def process(self, input) -> np.ndarray:
        return self._engine.process(input)

    def set_filter(self, ir) -> None:
        """exchange_filter(partition(ir, L, M)) (reference.cpp:335-338). The reference partitions on
        the caller's thread (a load spike); here the taps are staged and transformed (K4) on the
        device on a side stream overlapping the running hops, latched at the next process()."""
        e = self._engine
        s = partition(ir, e.hop(), e.partition_count())  # validation and M, as the reference
        e.exchange_ir(s.taps)
        e._filter = s

    def reset(self) -> None:
        self._engine.reset()

    def engine(self) -> TvolapEngine:
        return self._engine


# ---------------------------------------------------------------- comparison convolvers (§8f row 4)
@dataclass
class CrossfadeConfig:
    """CrossfadeConfig (reference.hpp:18-22): duration in samples (1 = hard switch), shape."""

    HANN = 0
    LINEAR = 1
    duration: int = 1
    shape: int = 0


class _CmpProcessor:
    """The reference's other streaming convolvers on the GPU (reference.hpp:53-200), through
    tvolap_cmp_* (include/tvolap_b200.h). process() takes hop() x channels() like the reference;
    process_hops() takes lanes x (n * hop())."""

    KIND = -1
    NAME = ""

    def __init__(self, ir, hop: int = 0, fade: Optional[CrossfadeConfig] = None, device: int = 0):
        h = np.asarray(ir, dtype=np.float64)
        if h.ndim == 1:
            h = h[:, None]
        taps = _f32(h.T) if h.size else np.zeros((max(h.shape[1], 1), 1), np.float32)
        fade = fade or CrossfadeConfig()
        self._h = C.c_void_p()
        _check(lib().tvolap_cmp_create(C.byref(self._h), device, self.KIND, h.shape[0], h.shape[1],
                                       taps.ctypes.data, max(h.shape[0], 1), hop, fade.duration, fade.shape))
        self.device = device

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tvolap_cmp_destroy(self._h)
            self._h = None

    def _geo(self):
        g = np.zeros(6, dtype=np.int64)
        _check(lib().tvolap_cmp_geometry(self._h, g.ctypes.data))
        return g

    def name(self) -> str:
        return self.NAME

    def hop(self) -> int:
        return int(self._geo()[0])

    def channels(self) -> int:
        return int(self._geo()[1])

    def latency(self) -> int:
        return int(self._geo()[2])

    def stream_delay(self) -> int:
        return int(self._geo()[3])

    def switching_latency(self) -> int:
        return int(self._geo()[4])

    def fading(self) -> bool:
        return bool(self._geo()[5])

    def channels_out(self) -> int:
        return self.channels()

    def process_hops(self, x) -> np.ndarray:
        """lanes x (n * hop) float32 -> same shape (n consecutive process() calls)."""
        xs = _f32(x)
        if xs.ndim != 2:
            raise InvalidInputError("process_hops expects lanes x samples")
        hop = self.hop()
        if xs.shape[1] % hop:
            raise InvalidSizeError("process_hops expects a whole number of hops")
        out = np.empty_like(xs)
        _check(lib().tvolap_cmp_process_hops(self._h, xs.ctypes.data, xs.shape[1], out.ctypes.data, out.shape[1],
                                             xs.shape[1] // hop))
        return out

    def process(self, input) -> np.ndarray:
        x = np.asarray(input, dtype=np.float64)
        if x.ndim == 1:
            x = x[:, None]
        if x.shape[0] != self.hop():
            raise InvalidSizeError("process() expects exactly one hop of input per call")
        if x.shape[1] != self.channels():
            raise InvalidInputError("input channel count does not match the filter")
        return self.process_hops(x.T).T.astype(np.float64)

    def set_filter(self, ir) -> None:
        h = np.asarray(ir, dtype=np.float64)
        if h.ndim == 1:
            h = h[:, None]
        t = _f32(h.T)
        _check(lib().tvolap_cmp_set_filter(self._h, t.ctypes.data, h.shape[0], h.shape[1], h.shape[0]))

    def reset(self) -> None:
        _check(lib().tvolap_cmp_reset(self._h))


class DirectProcessor(_CmpProcessor):
    """DirectProcessor "tdc" (reference.cpp:57-95): direct-form FIR, hard switch at hop boundaries."""

    KIND, NAME = 0, "tdc"

    def __init__(self, ir, hop: int, device: int = 0):
        super().__init__(ir, hop, device=device)


class CfTdcProcessor(_CmpProcessor):
    """CfTdcProcessor "cf-tdc" (reference.cpp:97-180): direct form, crossfaded filter switch."""

    KIND, NAME = 1, "cf-tdc"

    def __init__(self, ir, hop: int, fade: CrossfadeConfig, device: int = 0):
        super().__init__(ir, hop, fade=fade, device=device)

    def switch_filter(self, ir, fade: CrossfadeConfig) -> None:
        h = np.asarray(ir, dtype=np.float64)
        if h.ndim == 1:
            h = h[:, None]
        t = _f32(h.T)
        _check(lib().tvolap_cmp_switch_filter(self._h, t.ctypes.data, h.shape[0], h.shape[1], h.shape[0],
                                              fade.duration, fade.shape))


class OlaProcessor(_CmpProcessor):
    """OlaProcessor "ola" (reference.cpp:182-219): block = IR length, hop = block."""

    KIND, NAME = 2, "ola"

    def __init__(self, ir, device: int = 0):
        super().__init__(ir, 0, device=device)


class OlsProcessor(_CmpProcessor):
    """OlsProcessor "ols" (reference.cpp:221-255): block = IR length, hop = block."""

    KIND, NAME = 3, "ols"

    def __init__(self, ir, device: int = 0):
        super().__init__(ir, 0, device=device)


class WolaProcessor(_CmpProcessor):
    """WolaProcessor "wola" (reference.cpp:257-315): sqrt-Hann analysis/synthesis, hop = block / 2."""

    KIND, NAME = 4, "wola"

    def __init__(self, ir, device: int = 0):
        super().__init__(ir, 0, device=device)


def make_processor(name: str, ir, hop: int, device: int = 0):
    """make_processor (reference.cpp:345-363): "tdc", "cf-tdc" (cosine fade over one hop), "ola",
    "ols", "wola" (block forms ignore `hop`), "tvolap"."""
    if name == "tdc":
        return DirectProcessor(ir, hop, device=device)
    if name == "cf-tdc":
        return CfTdcProcessor(ir, hop, CrossfadeConfig(hop, CrossfadeConfig.HANN), device=device)
    if name == "ola":
        return OlaProcessor(ir, device=device)
    if name == "ols":
        return OlsProcessor(ir, device=device)
    if name == "wola":
        return WolaProcessor(ir, device=device)
    if name == "tvolap":
        return TvolapProcessor(ir, hop, device=device)
    raise InvalidConfigurationError(f"unknown algorithm: {name}")


# ---------------------------------------------------------------- frame adapter (frame_adapter.hpp)
class FrameAdapter:
    """Arbitrary host chunks -> exact hops (proj/include/tvolap/frame_adapter.hpp, frame_adapter.cpp:13-43).

    Buffers input until a full hop is available and returns output as it is produced, so the
    concatenated output equals feeding strict hops. Complete hops inside one pushed chunk go
    to the engine as a single multi-hop call (the hop-blocked kernel), which gives bit-identical
    results to one process() per hop.
    """

    def __init__(self, proc):
        self._proc = proc
        self._eng = proc.engine() if hasattr(proc, "engine") else proc
        self._hop = proc.hop()
        self._ch = proc.channels()
        self._staging = np.zeros((self._hop, self._ch), dtype=np.float32)
        self._fill = 0

    def buffered(self) -> int:
        return self._fill

    def push(self, chunk) -> np.ndarray:
        """frame_adapter.cpp:13-35: feed any number of frames (rows x channels)."""
        x = np.asarray(chunk, dtype=np.float32)
        if x.ndim == 1:
            x = x[:, None]
        if x.shape[1] != self._ch:
            raise InvalidInputError("adapter chunk channel count does not match the processor")
        hop, outs, pos = self._hop, [], 0
        if self._fill:  # complete the partial hop first
            take = min(hop - self._fill, x.shape[0])
            self._staging[self._fill:self._fill + take] = x[:take]
            self._fill += take
            pos = take
            if self._fill == hop:
                outs.append(self._proc.process(self._staging))
                self._fill = 0
        n_full = (x.shape[0] - pos) // hop
        if n_full:
            seg = x[pos:pos + n_full * hop]
            if n_full > 1:
                y = self._eng.process_hops(np.ascontiguousarray(seg.T))  # (lanes, n*hop)
                outs.append(y.T)
            else:
                outs.append(self._proc.process(seg))
            pos += n_full * hop
        rest = x.shape[0] - pos
        if rest:
            self._staging[:rest] = x[pos:]
            self._fill = rest
        if not outs:
            return np.zeros((0, self._eng.channels_out()), dtype=np.float32)
        return np.concatenate(outs, axis=0)

    def flush(self) -> np.ndarray:
        """frame_adapter.cpp:37-43: zero-pad the partial hop, if any, and process it."""
        if self._fill == 0:
            return np.zeros((0, self._eng.channels_out()), dtype=np.float32)
        self._staging[self._fill:] = 0.0
        self._fill = 0
        return self._proc.process(self._staging)
