"""Regenerate the golden fixtures in this directory from the fp64 CPU oracle.

The reference ships no golden vectors and cannot be built here (Eigen3 missing), so these
fixtures are oracle outputs on seeded inputs, committed so that (a) CPU tests catch any drift
of the oracle itself and (b) GPU tests compare the CUDA path against frozen numbers.

    python tests/golden/make_golden.py
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


if __name__ == "__main__":
    main()
