"""In-tree build of the native libraries (nvcc cross-compiles for sm_100a without a GPU).

Products (git-ignored, shipped to the GPU box with the repo snapshot):
  paper_2310_00319_b200/lib/libtvolap_b200.so    CUDA kernels + C-ABI (include/tvolap_b200.h)
  paper_2310_00319_b200/lib/libtvolap_workload.so host twin of the seeded generators
  paper_2310_00319_b200/lib/test_wrapper          C++ drop-in check of include/tvolap_b200.hpp
"""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_SOURCES = [CSRC / "tvolap_kernels.cu", CSRC / "tvolap_wide.cu", CSRC / "tvolap_engine.cu"]
CUDA_DEPS = CUDA_SOURCES + [CSRC / "tvolap_fft.cuh", CSRC / "tvolap_internal.cuh", CSRC / "workload.h",
                            INCLUDE / "tvolap_b200.h"]

LIB_CUDA = LIB / "libtvolap_b200.so"
LIB_WORKLOAD = LIB / "libtvolap_workload.so"
TEST_WRAPPER = LIB / "test_wrapper"


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd):
    subprocess.run([str(c) for c in cmd], check=True, cwd=ROOT)


def build(force: bool = False, verbose: bool = False) -> None:
    LIB.mkdir(exist_ok=True)
    if force or _stale(LIB_CUDA, CUDA_DEPS):
        # --fmad=false: no implicit multiply-add contraction, so the one-hop and hop-blocked
        # kernels (same operations, different code around them) round identically; every
        # intended FMA is an explicit fmaf().
        # host-only calls from device code compile to traps: make them errors
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Werror", "cross-execution-space-call",
               "-Xcompiler", "-fPIC", "-shared",
               "-I", INCLUDE, "-o", LIB_CUDA, *CUDA_SOURCES]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        _run(cmd)
    wsrc = [CSRC / "workload_host.cpp", CSRC / "workload.h"]
    if force or _stale(LIB_WORKLOAD, wsrc):
        _run(["g++", "-std=c++20", "-O3", "-fPIC", "-shared", "-pthread", "-o", LIB_WORKLOAD,
              CSRC / "workload_host.cpp"])
    tsrc = [ROOT / "tests" / "cpp" / "test_wrapper.cpp", INCLUDE / "tvolap_b200.hpp", INCLUDE / "tvolap_b200.h",
            LIB_CUDA]
    if (ROOT / "tests" / "cpp" / "test_wrapper.cpp").exists() and (force or _stale(TEST_WRAPPER, tsrc)):
        _run(["g++", "-std=c++17", "-O2", "-I", INCLUDE, "-o", TEST_WRAPPER,
              ROOT / "tests" / "cpp" / "test_wrapper.cpp", "-L", LIB, "-ltvolap_b200",
              f"-Wl,-rpath,{LIB}", "-Wl,-rpath,$ORIGIN"])


def build_variant(name: str, defines, verbose: bool = False) -> Path:
    """Diagnostic build of the CUDA library into lib/<name>/ (e.g. TVOLAP_PHASE_PROF for
    scripts/phase_prof.py). Never loaded by the product path."""
    out = LIB / name / "libtvolap_b200.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    if _stale(out, CUDA_DEPS):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Werror", "cross-execution-space-call",
              "-Xcompiler", "-fPIC", "-shared",
              *[f"-D{d}" for d in defines], "-I", INCLUDE, "-o", out, *CUDA_SOURCES])
    return out


REFERENCE = Path("/root/reference/proj")


def build_oracle(force: bool = False) -> None:
    """TEST INFRASTRUCTURE: the fp64 CPU oracle (oracle/Makefile) and, where /root/reference
    exists (this container, not the GPU box, which uses the prebuilt file), oracle/_ref: the
    reference's own hot-path sources compiled unmodified against the Eigen stand-in."""
    args = ["make", "-s", "-C", ROOT / "oracle"]
    if force:
        args.insert(2, "-B")
    _run(args)
    if (REFERENCE / "src" / "engine.cpp").exists():
        _run(args + ["ref"])


if __name__ == "__main__":
    build(force=True, verbose=True)
    build_oracle(force=True)
