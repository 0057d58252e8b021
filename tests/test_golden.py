"""Committed golden fixtures (tests/golden/golden_v{1,2}.npz, made by tests/golden/make_golden.py
from the REFERENCE's own hot-path sources, oracle/_ref): the restated oracle must keep reproducing
them bit for bit (CPU), and the CUDA path must match them within the north-star tolerance (GPU —
these are the reference's numbers on the GPU box, where /root/reference does not exist)."""
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2310_00319_b200 import drive
from paper_2310_00319_b200 import workload as W
from parity import TOL, oracle_config, rel_err

G = np.load(Path(__file__).resolve().parent / "golden" / "golden_v1.npz")
G2 = np.load(Path(__file__).resolve().parent / "golden" / "golden_v2.npz")


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


@pytest.mark.parametrize("name,key,hops,subset", [("C2", "c2_2x80", 80, [0, 63]), ("C3", "c3_2x2x300", 300, [0, 1023]),
                                                  ("C4", "c4_1x24", 24, [255])])
def test_oracle_reproduces_v2_goldens(name, key, hops, subset):
    y = oracle_config(W.CONFIGS[name], hops, subset=subset, which="port")
    assert np.array_equal(y.astype(np.float32), G2[key])


@pytest.mark.gpu
@pytest.mark.parametrize("name,key,hops,lanes", [("C2", "c2_2x80", 80, [0, 63]), ("C3", "c3_2x2x300", 300, [0, 1, 2046, 2047]),
                                                 ("C4", "c4_1x24", 24, [255])])
def test_gpu_matches_v2_goldens(name, key, hops, lanes):
    """Full lane count of the config on the GPU; the golden lanes compared with the reference's output."""
    _, y = drive.run_host(W.CONFIGS[name], hops)
    assert rel_err(y[lanes], G2[key].astype(np.float64)) <= TOL
