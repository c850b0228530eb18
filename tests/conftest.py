import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")
    config.addinivalue_line("markers", "slow: full-size (BASELINE config) parity checks")


@pytest.fixture(scope="session")
def adaln_golden():
    return np.load(GOLDEN / "adaln_golden.npz")


@pytest.fixture(scope="session")
def sampler_golden():
    return json.loads((GOLDEN / "sampler_golden.json").read_text())


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda", 0)


def max_rel_err(a, r) -> float:
    """The reference's tolerance convention max|a-r| / max|r| (adaln/__init__.py:217-219)."""
    a = np.asarray(a, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    return float(np.abs(a - r).max()) / max(float(np.abs(r).max()), 1e-12)
