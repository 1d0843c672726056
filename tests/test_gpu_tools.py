"""GPU: tools/evolve.py writes the reference's evolve CSV (step,time,energy,
gauss_residual with %.17g; reference tools/sfeec_main.cpp:193-215)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("args", [["--config", "tet8", "--steps", "40", "--diag-every", "10"],
                                  ["--config", "yee", "--n", "12", "--steps", "50",
                                   "--diag-every", "10"]])
def test_evolve_csv(args, tmp_path):
    out = tmp_path / "e.csv"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "evolve.py"), *args, "--out",
                    str(out)], check=True, timeout=300)
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "step,time,energy,gauss_residual"
    rows = np.array([[float(v) for v in l.split(",")] for l in lines[1:]])
    assert rows.shape[0] == 1 + int(args[args.index("--steps") + 1]) // 10
    assert np.all(rows[:, 2] > 0)
    assert np.all(rows[:, 3] <= 1e-10 * max(1.0, rows[:, 2].max()))
