import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


def _ensure_built():
    """Build the product library and the C checker if they are missing."""
    import subprocess
    lib = os.path.join(ROOT, "paper_2301_01753_b200", "libsfeec_b200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j8"], cwd=os.path.join(ROOT, "paper_2301_01753_b200",
                                                              "csrc"), check=True)
    port = os.path.join(ROOT, "oracle", "_build", "libsfeec_oracle.so")
    if not os.path.exists(port):
        subprocess.run(["make", "-s", "_build/libsfeec_oracle.so"],
                       cwd=os.path.join(ROOT, "oracle"), check=True)


_ensure_built()


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name))
    return load


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
