import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
# the oracle's OpenMP regions are tiny at test sizes: one thread is fastest
os.environ.setdefault("OMP_NUM_THREADS", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden_tables():
    return np.load(GOLDEN / "tables_small.npz")


@pytest.fixture(scope="session")
def golden_hashes():
    return json.loads((GOLDEN / "tables_hash.json").read_text())


@pytest.fixture(scope="session")
def golden_rhs():
    return np.load(GOLDEN / "rhs_cases.npz")


@pytest.fixture(scope="session")
def golden_traj():
    return np.load(GOLDEN / "traj.npz"), json.loads((GOLDEN / "traj.json").read_text())


@pytest.fixture(scope="session")
def golden_long():
    path = GOLDEN / "traj_long.npz"
    if not path.exists():
        pytest.skip("long golden fixture not generated")
    return np.load(path), json.loads((GOLDEN / "traj_long.json").read_text())


def gpu_available() -> bool:
    try:
        from paper_1012_4382_b200 import _native
        return _native.device_count() > 0
    except Exception:
        return False
