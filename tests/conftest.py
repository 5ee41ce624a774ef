"""Test configuration: the ``gpu`` marker and shared fixtures.

``-m "not gpu"``: oracle vs golden fixtures, host logic, ABI symbol checks,
multi-rank (gloo) sharding - runs on the CPU-only build container.
``-m gpu``: parity of the CUDA path (through the C ABI) against the oracle and
the golden fixtures - runs on a B200.
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libuqg.so")


@pytest.fixture(scope="session")
def pcg_golden():
    with np.load(GOLDEN / "pcg_cases.npz") as z:
        d = {k: z[k] for k in z.files}
    n = int(d["n_cases"])
    return [{k[len(f"c{c}_"):]: v for k, v in d.items() if k.startswith(f"c{c}_")} for c in range(n)]


@pytest.fixture(scope="session")
def special_golden():
    with np.load(GOLDEN / "special_cases.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def grouping_golden():
    return json.loads((GOLDEN / "grouping.json").read_text())


@pytest.fixture(scope="session")
def c1_golden():
    return json.loads((GOLDEN / "c1_adaptive.json").read_text())


@pytest.fixture(scope="session")
def c2_golden():
    return json.loads((GOLDEN / "c2_group.json").read_text())


@pytest.fixture(scope="session")
def eigen_golden():
    with np.load(GOLDEN / "eigen.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def fv2d_golden():
    with np.load(GOLDEN / "fv2d_small.npz") as z:
        return {k: z[k] for k in z.files}
