"""The C++ drop-in API (include/sfeec/*.hpp, reference-compatible signatures):
compiles on CPU; its reference-style test program passes on the GPU."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

CXX_DIR = os.path.join(ROOT, "tests", "cxx")


def _build():
    subprocess.run(["make", "-s", "test_dropin"], cwd=CXX_DIR, check=True)
    return os.path.join(CXX_DIR, "test_dropin")


def test_dropin_compiles_against_reference_style_headers():
    exe = _build()
    assert os.access(exe, os.X_OK)


@pytest.mark.gpu
def test_dropin_program_passes_on_device():
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
