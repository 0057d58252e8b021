import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: longer CPU oracle runs")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the native libraries in-tree once per session (no-op when up to date)."""
    from paper_2310_00319_b200 import _build

    _build.build()
    _build.build_oracle()
    yield


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(autouse=True)
def _default_tuning_reset():
    """Tests that set process-wide default tuning (tvolap_set_default_tuning) leave none behind."""
    yield
    import paper_2310_00319_b200.tvolap as T

    if T._lib is not None:
        T.reset_default_tuning()
