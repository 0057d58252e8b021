"""Regenerate the golden fixtures in this directory from THE REFERENCE ITSELF.

The reference ships no golden vectors. Its hot path (proj/src/{spectral,partition,engine}.cpp)
is compiled unmodified from /root/reference against a minimal Eigen stand-in into
oracle/_ref/libtvolap_ref.so (oracle/Makefile `ref`), and every fixture here is that library's
output on seeded inputs (the restated oracle produces the same bits: tests/test_ref_pin.py).
Committed so that (a) CPU tests catch drift of the oracle, and (b) GPU tests compare the CUDA
path against frozen reference numbers on the GPU box, where /root/reference does not exist.

    python tests/golden/make_golden.py      (needs /root/reference, i.e. this container)
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))

import oracle as O  # noqa: E402
from paper_2310_00319_b200 import workload as W  # noqa: E402
from parity import oracle_config  # noqa: E402


def main():
    assert O.ref_available(), "build oracle/_ref first (make -C oracle ref)"
    with O.using("ref"):
        v1()
        v2()


def v1():
    # 1. spectral: forward_real of a seeded 64-sample block, inverse of it
    x = W.white(W.CONFIGS["C1"], 7, 1, 0, 64, dtype=np.float64)[0]
    fr = O.forward_real(x)
    # 2. partition spectra of a seeded 300-tap IR at L = 16, min_partitions 12
    ir = W.white(W.CONFIGS["C1"], 8, 1, 0, 300, dtype=np.float64)[0]
    ps = O.partition(ir, 16, 12).spectra()[0]
    # 3. C1 (1 lane, L=128, M=32, two IRs alternating every 64 blocks): first 200 hops
    c1 = oracle_config(W.CONFIGS["C1"], 200)
    # 4. C5 geometry (L=32, M=512 bank, per-hop choice): 2 lanes x 1030 hops (ring wrapped)
    c5 = oracle_config(W.CONFIGS["C5"], 1030, subset=[0, 4095])
    np.savez_compressed(HERE / "golden_v1.npz", fr_in=x, fr_out=fr, part_ir=ir, part_spectra=ps,
                        c1_200=c1.astype(np.float32), c5_2x1030=c5.astype(np.float32))
    print("wrote", HERE / "golden_v1.npz")


def v2():
    """The other BASELINE configs' geometries and switch schedules (prefixes)."""
    c2 = oracle_config(W.CONFIGS["C2"], 80, subset=[0, 63])            # fresh IR every 16 hops
    c3 = oracle_config(W.CONFIGS["C3"], 300, subset=[0, 1023])         # 2 sources x 2 ears, bank choice per hop
    c4 = oracle_config(W.CONFIGS["C4"], 24, subset=[255])              # fresh IR every 8 hops, L=512 M=256
    np.savez_compressed(HERE / "golden_v2.npz", c2_2x80=c2.astype(np.float32), c3_2x2x300=c3.astype(np.float32),
                        c4_1x24=c4.astype(np.float32))
    print("wrote", HERE / "golden_v2.npz")


if __name__ == "__main__":
    main()
