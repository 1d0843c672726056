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


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("extra", [["--config", "tet16"], ["--config", "tet16", "--strong"]])
def test_bench_two_ranks_over_ipc(extra):
    """The driver's N > 1 launch of bench.py (torchrun, one process per rank)
    with the host-synchronised CUDA-IPC transport, both ranks on this GPU: the
    multi-rank bench flow end to end (rendezvous, id broadcast, per-rank slab
    assembly, distributed CFL, max-over-ranks timing, one JSON line). A
    functional check; the numbers are not scaling numbers."""
    import json
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "20", "--warmup", "3",
           "--transport", "ipc", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 20 and d["value"] > 0
    assert d["scaling"] == ("strong" if "--strong" in extra else "weak")
    n1, n2 = 26416, 50688  # tet16's DOFs
    if "--strong" in extra:  # the 16^3 mesh split in two
        assert d["value"] == pytest.approx((n1 + n2) * 20 / (d["ms_per_step"] * 20e-3))
    # (white-noise A: a bounded oscillation of the discrete energy, not a blow-up)
    assert abs(d["physics"]["rel_energy_change"]) < 0.25
