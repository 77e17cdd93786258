import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and libpffmg.so")
    config.addinivalue_line("markers", "slow: long-running")


class Golden:
    """Lazy view of one tests/golden/*.npz file."""

    def __init__(self, name):
        self.path = os.path.join(GOLDEN, f"{name}.npz")
        self._z = None

    @property
    def z(self):
        if self._z is None:
            self._z = np.load(self.path)
        return self._z

    def __getitem__(self, key):
        return self.z[key]

    def has(self, key):
        return key in self.z.files

    def exists(self):
        return os.path.exists(self.path)


@pytest.fixture(scope="session")
def golden():
    return {n: Golden(n) for n in ("meshes", "operator", "operator_band", "transfers", "multigrid", "multigrid_miehe", "qoi", "boundary", "configs", "configs_full", "newton", "scenarios", "krylov")}


def rel_err(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
