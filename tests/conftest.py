import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def golden():
    class G:
        def __init__(self):
            self._cache = {}

        def __call__(self, name):
            if name not in self._cache:
                self._cache[name] = np.load(GOLDEN / f"{name}.npz")
            return self._cache[name]
    return G()


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def lib():
    """The product's C-ABI library (GPU tests only)."""
    if not cuda_ok():
        pytest.skip("no CUDA device")
    from paper_2605_28691_b200 import _lib
    return _lib.lib()


# ---- parity report: tests record max-abs / relative-L2 errors per tensor; with OSP_PARITY_OUT set
# the session writes them as JSON (profiles/rNN_parity.json is a committed copy of one run)
PARITY: dict = {}


@pytest.fixture(scope="session")
def parity_record():
    def rec(case: str, entry: dict):
        PARITY[case] = entry
    return rec


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("OSP_PARITY_OUT")
    if out and PARITY:
        Path(out).parent.mkdir(parents=True, exist_ok=True)
        Path(out).write_text(json.dumps(PARITY, indent=1, sort_keys=True))
