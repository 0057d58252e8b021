"""Committed golden fixtures (tests/golden/golden_v1.npz, made by tests/golden/make_golden.py
from the fp64 oracle): the oracle must keep reproducing them (CPU), and the CUDA path must match
them within the north-star tolerance (GPU)."""
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2310_00319_b200 import drive
from paper_2310_00319_b200 import workload as W
from parity import TOL, oracle_config, rel_err

G = np.load(Path(__file__).resolve().parent / "golden" / "golden_v1.npz")


def test_oracle_reproduces_spectral_goldens():
    assert np.array_equal(O.forward_real(G["fr_in"]), G["fr_out"])
    assert np.array_equal(O.partition(G["part_ir"], 16, 12).spectra()[0], G["part_spectra"])


def test_oracle_reproduces_c1_prefix():
    assert np.array_equal(oracle_config(W.CONFIGS["C1"], 64).astype(np.float32), G["c1_200"][:, : 64 * 128])


def test_workload_generators_unchanged():
    assert np.array_equal(W.white(W.CONFIGS["C1"], 7, 1, 0, 64, dtype=np.float64)[0], G["fr_in"])


@pytest.mark.gpu
def test_gpu_matches_golden_c1():
    _, y = drive.run_host(W.CONFIGS["C1"], 200)
    assert rel_err(y, G["c1_200"].astype(np.float64)) <= TOL


@pytest.mark.gpu
def test_gpu_matches_golden_c5_full_lane_count():
    cfg = W.CONFIGS["C5"]
    _, y = drive.run_host(cfg, 1030)
    assert rel_err(y[[0, 4095]], G["c5_2x1030"].astype(np.float64)) <= TOL


@pytest.mark.gpu
def test_gpu_spectral_goldens():
    from paper_2310_00319_b200 import tvolap as T

    fr = T.forward_real(G["fr_in"].astype(np.float32))
    assert np.abs(fr - G["fr_out"]).max() <= 1e-5 * np.abs(G["fr_out"]).max()
    ps = T.partition(G["part_ir"].astype(np.float32), 16, 12).spectra()[0]
    assert np.abs(ps - G["part_spectra"]).max() <= 1e-5 * np.abs(G["part_spectra"]).max()
