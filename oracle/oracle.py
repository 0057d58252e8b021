"""TEST INFRASTRUCTURE ONLY — ctypes view of the fp64 CPU oracle (oracle/liboracle.so).

The oracle restates the reference hot path (proj/src/spectral.cpp, partition.cpp,
engine.cpp) in plain C++; see oracle/tvolap_oracle.cpp for the line citations.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this
module. The product package never does.

`using("ref")` switches the same API onto oracle/_ref/libtvolap_ref.so: the
reference's OWN spectral/partition/engine sources compiled unmodified against a
minimal Eigen stand-in (oracle/Makefile `ref`, oracle/ref_harness.cpp). That is
what pins the restatement (tests/test_ref_pin.py) and what bench.py's reference
arm times. The comparison convolvers and direct_convolve exist only in the port.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from contextlib import contextmanager
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_SO = HERE / "liboracle.so"
_REF_SO = HERE / "_ref" / "libtvolap_ref.so"
_libs = {}
_which = "port"
_lib = None  # the port, once loaded (kept for the __del__ guards below)


class OracleError(ValueError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def ref_available() -> bool:
    """oracle/_ref/libtvolap_ref.so exists (built here from /root/reference, shipped to the box)."""
    return _REF_SO.exists()


@contextmanager
def using(which):
    """Run the enclosed oracle calls on "port" (the restatement) or "ref" (the reference itself)."""
    global _which
    prev, _which = _which, which
    try:
        yield
    finally:
        _which = prev


def lib():
    global _lib
    if _which not in _libs:
        path = _SO if _which == "port" else _REF_SO
        if _which == "port" and not _SO.exists():
            build()
        if not path.exists():
            raise OracleError(3, f"{path} not built (oracle/Makefile target `ref` needs /root/reference)")
        L = C.CDLL(str(path))
        vp, lg, ip = C.c_void_p, C.c_long, C.c_int
        L.orc_last_error.restype = C.c_char_p
        L.orc_forward_real.argtypes = [lg, vp, vp]
        L.orc_inverse_real.argtypes = [lg, lg, vp, vp]
        L.orc_mac.argtypes = [lg, lg, lg, lg, lg, lg, vp, vp, vp, vp]
        L.orc_hann_window.argtypes = [lg, vp]
        L.orc_partition.argtypes = [vp, lg, lg, lg, lg, C.POINTER(ip)]
        L.orc_partition.restype = vp
        L.orc_set_free.argtypes = [vp]
        for f in ("orc_set_partition_count", "orc_set_channels", "orc_set_hop", "orc_set_source_length"):
            getattr(L, f).argtypes = [vp]
            getattr(L, f).restype = lg
        L.orc_set_gain.argtypes = [vp]
        L.orc_set_gain.restype = C.c_double
        L.orc_set_spectra.argtypes = [vp, vp]
        L.orc_reassemble.argtypes = [vp, vp]
        L.orc_engine_create.argtypes = [vp, C.POINTER(ip)]
        L.orc_engine_create.restype = vp
        L.orc_engine_free.argtypes = [vp]
        L.orc_engine_process.argtypes = [vp, vp, lg, lg, lg, vp, lg]
        L.orc_engine_exchange.argtypes = [vp, vp]
        L.orc_engine_reset.argtypes = [vp]
        L.orc_engine_geometry.argtypes = [vp, vp]
        L.orc_engine_op_counts.argtypes = [vp, vp]
        if hasattr(L, "orc_direct_convolve"):
            L.orc_direct_convolve.argtypes = [vp, lg, vp, lg, vp]
        L.orc_run_workload.argtypes = [lg, lg, lg, lg, lg, vp, lg, ip, vp, lg, lg, lg, vp, vp, vp, lg, ip,
                                       C.POINTER(ip)]
        L.orc_run_workload.restype = C.c_double
        _libs[_which] = L
        if _which == "port":
            _lib = L
    return _libs[_which]


def _chk(rc, L=None):
    if rc:
        raise OracleError(rc, (L or lib()).orc_last_error().decode())


def _d(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def forward_real(x):
    x = _d(x)
    out = np.empty((x.size // 2 + 1, 2))
    _chk(lib().orc_forward_real(x.size, x.ctypes.data if x.size else None, out.ctypes.data))
    return out[:, 0] + 1j * out[:, 1]


def inverse_real(bins, n=None):
    b = np.asarray(bins, dtype=np.complex128)
    n = 2 * (b.size - 1) if n is None else n
    inter = np.ascontiguousarray(np.stack([b.real, b.imag], -1))
    out = np.empty(max(n, 0))
    _chk(lib().orc_inverse_real(n, b.size, inter.ctypes.data, out.ctypes.data if out.size else None))
    return out


def mac(acc, a, b, n=None):
    acc, a, b = (np.asarray(v, dtype=np.complex128) for v in (acc, a, b))
    ns = [2 * (v.size - 1) if n is None else n for v in (acc, a, b)]
    st = [np.ascontiguousarray(np.stack([v.real, v.imag], -1)) for v in (acc, a, b)]
    out = np.empty_like(st[0])
    _chk(lib().orc_mac(ns[0], ns[1], ns[2], acc.size, a.size, b.size, st[0].ctypes.data, st[1].ctypes.data,
                       st[2].ctypes.data, out.ctypes.data))
    return out[:, 0] + 1j * out[:, 1]


def hann_window(hop):
    w = np.empty(max(2 * hop, 0))
    _chk(lib().orc_hann_window(hop, w.ctypes.data if w.size else None))
    return w


class FilterSet:
    """partition(ir, hop, min_partitions) result (partition.hpp:21-32)."""

    def __init__(self, ir, hop, min_partitions=1):
        h = np.asarray(ir, dtype=np.float64)
        if h.ndim == 1:
            h = h[:, None]
        taps = np.ascontiguousarray(h.T)
        st = C.c_int()
        ptr = taps.ctypes.data if taps.size else None
        self._L = lib()
        self._h = self._L.orc_partition(ptr, h.shape[0], h.shape[1] if h.ndim == 2 else 0, hop, min_partitions,
                                        C.byref(st))
        _chk(st.value, self._L)

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.orc_set_free(self._h)

    @property
    def partition_count(self):
        return self._L.orc_set_partition_count(self._h)

    @property
    def channels(self):
        return self._L.orc_set_channels(self._h)

    @property
    def hop(self):
        return self._L.orc_set_hop(self._h)

    @property
    def source_length(self):
        return self._L.orc_set_source_length(self._h)

    @property
    def normalization_gain(self):
        return self._L.orc_set_gain(self._h)

    def transform_length(self):
        return 4 * self.hop

    def padded_length(self):
        return 2 * self.hop * self.partition_count

    def spectra(self):
        out = np.empty((self.channels, self.partition_count, 2 * self.hop + 1, 2))
        self._L.orc_set_spectra(self._h, out.ctypes.data)
        return out[..., 0] + 1j * out[..., 1]

    def reassemble(self):
        out = np.empty((self.channels, 2 * self.hop * self.partition_count))
        _chk(self._L.orc_reassemble(self._h, out.ctypes.data), self._L)
        return out.T.copy()  # (taps, channels), like ImpulseResponse


def partition(ir, hop, min_partitions=1):
    return FilterSet(ir, hop, min_partitions)


class Engine:
    """TvolapEngine (engine.hpp:33-94), fp64."""

    def __init__(self, filter_set):
        st = C.c_int()
        self._set = filter_set
        self._L = lib()
        self._h = self._L.orc_engine_create(filter_set._h if filter_set is not None else None, C.byref(st))
        _chk(st.value, self._L)

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.orc_engine_free(self._h)

    def _geo(self):
        g = np.empty(7, dtype=np.int64)
        self._L.orc_engine_geometry(self._h, g.ctypes.data)
        return g

    def hop(self):
        return int(self._geo()[0])

    def channels(self):
        return int(self._geo()[1])

    def partition_count(self):
        return int(self._geo()[2])

    def delay_line_depth(self):
        return int(self._geo()[3])

    def latency(self):
        return int(self._geo()[4])

    def switching_latency(self):
        return int(self._geo()[5])

    def stream_delay(self):
        return int(self._geo()[6])

    def process(self, x):
        x = np.asarray(x, dtype=np.float64)
        if x.ndim == 1:
            x = x[:, None]
        rows, cols = x.shape
        xf = np.ascontiguousarray(x.T)
        out = np.empty((max(cols, 1), max(rows, 1)))
        _chk(self._L.orc_engine_process(self._h, xf.ctypes.data if xf.size else None, max(rows, 1), rows, cols,
                                        out.ctypes.data, max(rows, 1)), self._L)
        return out.T.copy()

    def exchange_filter(self, filter_set):
        self._next = filter_set
        _chk(self._L.orc_engine_exchange(self._h, filter_set._h if filter_set is not None else None), self._L)

    def reset(self):
        self._L.orc_engine_reset(self._h)

    def op_counts(self):
        c = np.empty(3, dtype=np.uint64)
        self._L.orc_engine_op_counts(self._h, c.ctypes.data)
        return tuple(int(v) for v in c)


def direct_convolve(x, h):
    """reference.cpp:10-32 (single channel)."""
    x, h = _d(x), _d(h)
    out = np.empty(x.size + h.size - 1)
    lib().orc_direct_convolve(x.ctypes.data, x.size, h.ctypes.data, h.size, out.ctypes.data)
    return out


def stream_through(eng, x, n_out):
    """test_engine.cpp:28-38: feed hop by hop plus zero hops; drop the stream delay."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    hop = eng.hop()
    total = n_out + eng.stream_delay()
    calls = -(-total // hop)
    padded = np.zeros((calls * hop, x.shape[1]))
    padded[: x.shape[0]] = x
    out = np.empty((calls * hop, eng.channels_out() if hasattr(eng, "channels_out") else x.shape[1]))
    for i in range(calls):
        out[i * hop:(i + 1) * hop] = eng.process(padded[i * hop:(i + 1) * hop])
    return out[eng.stream_delay(): eng.stream_delay() + n_out]


def run_workload(hop, min_partitions, sources, ears, n_hops, x, mode, fresh_ir=None, period=1, bank_ir=None,
                 schedule=None, want_output=True, threads=1):
    """Threaded drive() of a whole workload (see orc_run_workload). Returns (seconds, out or None).

    x: (sources, >= n_hops*hop) float64; fresh_ir: (n_switch, sources, ears, ir_len);
    bank_ir: (n_bank, ears, ir_len); schedule: (n_hops, sources) int32.
    """
    x = _d(x)
    ir_len = fresh_ir.shape[-1] if mode == 0 else bank_ir.shape[-1]
    fi = _d(fresh_ir) if fresh_ir is not None else None
    bi = _d(bank_ir) if bank_ir is not None else None
    sc = np.ascontiguousarray(schedule, dtype=np.int32) if schedule is not None else None
    n_bank = bi.shape[0] if bi is not None else 0
    out = np.empty((sources * ears, n_hops * hop)) if want_output else None
    st = C.c_int()
    secs = lib().orc_run_workload(hop, min_partitions, sources, ears, n_hops, x.ctypes.data, x.shape[1], mode,
                                  fi.ctypes.data if fi is not None else None, ir_len, period, n_bank,
                                  bi.ctypes.data if bi is not None else None,
                                  sc.ctypes.data if sc is not None else None,
                                  out.ctypes.data if out is not None else None, n_hops * hop, threads, C.byref(st))
    _chk(st.value)
    return secs, out


# ----------------------------------------------------------------- comparison convolvers
# reference.cpp:34-363: "tdc", "cf-tdc", "ola", "ols", "wola".
KINDS = {"tdc": 0, "cf-tdc": 1, "ola": 2, "ols": 3, "wola": 4}
HANN, LINEAR = 0, 1


def _cmp_sigs(L):
    vp, lg, ip = C.c_void_p, C.c_long, C.c_int
    if getattr(L, "_cmp_ready", False):
        return L
    L.orc_cmp_create.argtypes = [ip, vp, lg, lg, lg, lg, ip, C.POINTER(ip)]
    L.orc_cmp_create.restype = vp
    L.orc_cmp_free.argtypes = [vp]
    L.orc_cmp_process.argtypes = [vp, vp, lg, lg, lg, vp, lg]
    L.orc_cmp_set_filter.argtypes = [vp, vp, lg, lg]
    L.orc_cmp_switch_filter.argtypes = [vp, vp, lg, lg, lg, ip]
    L.orc_cmp_reset.argtypes = [vp]
    L.orc_cmp_geometry.argtypes = [vp, vp]
    L._cmp_ready = True
    return L


def _taps(ir):
    h = np.asarray(ir, dtype=np.float64)
    if h.ndim == 1:
        h = h[:, None]
    return h, np.ascontiguousarray(h.T)


class Processor:
    """A reference comparison convolver (reference.hpp:53-200): process() takes hop() x channels()."""

    def __init__(self, name, ir, hop=0, fade_duration=1, fade_shape=HANN):
        L = _cmp_sigs(lib())
        h, t = _taps(ir)
        st = C.c_int()
        self.name = name
        self._h = L.orc_cmp_create(KINDS[name], t.ctypes.data if t.size else None, h.shape[0], h.shape[1], hop,
                                   fade_duration, fade_shape, C.byref(st))
        _chk(st.value)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_cmp_free(self._h)
            self._h = None

    def _geo(self):
        g = np.zeros(6, dtype=np.int64)
        lib().orc_cmp_geometry(self._h, g.ctypes.data)
        return g

    def hop(self):
        return int(self._geo()[0])

    def channels(self):
        return int(self._geo()[1])

    def latency(self):
        return int(self._geo()[2])

    def stream_delay(self):
        return int(self._geo()[3])

    def switching_latency(self):
        return int(self._geo()[4])

    def fading(self):
        return bool(self._geo()[5])

    def process(self, x):
        x = np.asarray(x, dtype=np.float64)
        if x.ndim == 1:
            x = x[:, None]
        rows, cols = x.shape
        xf = np.ascontiguousarray(x.T)
        out = np.empty((max(cols, 1), max(rows, 1)))
        _chk(lib().orc_cmp_process(self._h, xf.ctypes.data if xf.size else None, max(rows, 1), rows, cols,
                                   out.ctypes.data, max(rows, 1)))
        return out.T.copy()

    def set_filter(self, ir):
        h, t = _taps(ir)
        _chk(lib().orc_cmp_set_filter(self._h, t.ctypes.data, h.shape[0], h.shape[1]))

    def switch_filter(self, ir, fade_duration, fade_shape=HANN):
        h, t = _taps(ir)
        _chk(lib().orc_cmp_switch_filter(self._h, t.ctypes.data, h.shape[0], h.shape[1], fade_duration, fade_shape))

    def reset(self):
        lib().orc_cmp_reset(self._h)


def make_processor(name, ir, hop):
    """reference.cpp:345-363: the factory (cf-tdc fades over one hop, Hann-complementary)."""
    if name == "tdc":
        return Processor("tdc", ir, hop)
    if name == "cf-tdc":
        return Processor("cf-tdc", ir, hop, fade_duration=hop)
    if name in ("ola", "ols", "wola"):
        return Processor(name, ir)
    if name == "tvolap":
        return Engine(partition(np.asarray(ir, dtype=np.float64), hop))
    raise OracleError(3, "unknown algorithm: " + name)
