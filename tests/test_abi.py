"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/tvolap_b200.h declares, and — without a GPU — fails loudly
instead of falling back to a CPU path."""
import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import gpu_available
from paper_2310_00319_b200 import tvolap as T

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "tvolap_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(tvolap_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_match_binding_list():
    assert declared_symbols() == sorted(T.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(T._LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", str(T._LIB_PATH)], capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", nm), f"{name} not exported"


def test_library_is_built_for_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(T._LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_header_compiles_as_c():
    src = f'#include "{HEADER}"\nint main(void) {{ return TVOLAP_OK; }}\n'
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-x", "c", "-", "-fsyntax-only"], input=src,
                       text=True, capture_output=True)
    assert r.returncode == 0, r.stderr


def test_status_codes_match_oracle_numbering():
    text = HEADER.read_text()
    codes = dict(re.findall(r"#define (TVOLAP_\w+) (\d+)", text))
    assert codes["TVOLAP_ERR_INVALID_SIZE"] == "1" and codes["TVOLAP_ERR_INVALID_INPUT"] == "2"
    assert codes["TVOLAP_ERR_INVALID_CONFIGURATION"] == "3" and codes["TVOLAP_ERR_INCOMPATIBLE_FILTER"] == "4"
    assert codes["TVOLAP_ERR_INVALID_SPECTRUM"] == "5"


def test_argument_validation_without_device():
    """Shape/size errors are raised before any device work, with the reference's classes."""
    with pytest.raises(T.InvalidSizeError):
        T.forward_real(np.zeros(12))
    with pytest.raises(T.InvalidSizeError):
        T.hann_window(1)
    with pytest.raises(T.InvalidInputError):
        T.partition(np.zeros((0, 1)), 64)
    with pytest.raises(T.InvalidSizeError):
        T.partition(np.ones(10), 24)
    h = ctypes.c_void_p()
    ir = np.ones(10, np.float32)
    assert T.lib().tvolap_create(ctypes.byref(h), 0, 24, 1, 10, ir.ctypes.data, 1) == 1
    assert T.lib().tvolap_create(ctypes.byref(h), 0, 64, 1, 0, ir.ctypes.data, 1) == 2
    # comparison convolvers (§8f row 4): the reference's constructor checks, before any device work
    c = ctypes.c_void_p()
    assert T.lib().tvolap_cmp_create(ctypes.byref(c), 0, 2, 100, 1, ir.ctypes.data, 100, 0, 1, 0) == 1  # ola: 2^k
    assert T.lib().tvolap_cmp_create(ctypes.byref(c), 0, 0, 10, 1, ir.ctypes.data, 10, 0, 1, 0) == 3  # tdc: hop < 1
    assert T.lib().tvolap_cmp_create(ctypes.byref(c), 0, 1, 10, 1, ir.ctypes.data, 10, 8, 0, 0) == 3  # fade < 1
    assert T.lib().tvolap_cmp_create(ctypes.byref(c), 0, 9, 10, 1, ir.ctypes.data, 10, 8, 1, 0) == 3  # kind
    with pytest.raises(T.InvalidSizeError):
        T.OlaProcessor(np.ones(100))


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(T.CudaError, match="no CPU fallback|CUDA"):
        T.TvolapEngine(T.partition(np.ones(100), 64))
    with pytest.raises(T.CudaError):
        T.forward_real(np.ones(16))


def test_cpp_wrapper_compiles():
    """include/tvolap_b200.hpp (the header-only C++ drop-in) builds against the C-ABI."""
    exe = ROOT / "paper_2310_00319_b200" / "lib" / "test_wrapper"
    assert exe.exists()


def test_tuning_table_without_device():
    """Every A/B knob is a named tuning key (no environment variables); defaults round-trip and
    bad keys / values fail with INVALID_INPUT — all host-side, no GPU needed."""
    keys = T.tuning_keys()
    for k in ("wide", "bank_pass", "bank_pass_mb", "k4_side", "k4_stream", "pdl", "k4_warp", "jh", "pb"):
        assert k in keys
    T.set_default_tuning("bank_pass", 0)
    T.set_default_tuning("pdl", 0)
    T.reset_default_tuning()
    with pytest.raises(T.InvalidInputError):
        T.set_default_tuning("no_such_knob", 1)
    with pytest.raises(T.InvalidInputError):
        T.set_default_tuning("wide", 9)
    assert T.lib().tvolap_set_tuning(None, b"wide", 1) != 0


def test_no_environment_reads_in_the_library():
    """Kernel / geometry choices are not steered by the environment."""
    src = "".join(p.read_text() for p in (ROOT / "paper_2310_00319_b200" / "csrc").glob("*.cu"))
    assert "getenv" not in src
