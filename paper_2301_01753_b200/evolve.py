"""The reference's `evolve` driver on the device.

`cmd_evolve` (reference tools/sfeec_main.cpp:151-215) steps a SplitScheme
and writes a CSV history `step,time,energy,gauss_residual` (printf
"%d,%.17g,%.17g,%.17g"): a row at step 0, then every `diag_every` steps and
at the last step. Here the state stays in HBM for the whole run: the
diagnostics are the device reductions (sfeec_dev_energy /
sfeec_dev_gauss_residual, dynamics.cpp:92-112) and only scalars cross PCIe.
Checkpoints save / restore a FieldState (formulation, first, e, time).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .inputs import uniform
from .scheme import FieldState, Formulation, SparseOperator, SplitScheme, make_state


def evolve_initial_state(c: SparseOperator, init_seed: int,
                         formulation: Formulation = Formulation.BE) -> FieldState:
    """cmd_evolve's initial state (sfeec_main.cpp:187-196): a and e drawn in that
    order from one Rng(init_seed) stream, uniform(-1, 1); BE starts from b = C a."""
    n1 = c.cols
    ae = uniform(init_seed, 2 * n1)
    a, e = ae[:n1].copy(), ae[n1:].copy()
    if Formulation(formulation) == Formulation.BE:
        from .configs import spmv
        return make_state(Formulation.BE, spmv(c, a), e)
    return make_state(Formulation.AE, a, e)


def _row(step: int, time: float, energy: float, gauss: float) -> str:
    return f"{step},{time:.17g},{energy:.17g},{gauss:.17g}\n"


def evolve(scheme: SplitScheme, state: FieldState, steps: int, diag_every: int = 1,
           out: str | None = None) -> str:
    """Advance `steps` steps from `state` with the history of cmd_evolve; the
    CSV text is returned (and written to `out`). The final state stays
    resident in the scheme (scheme.fetch())."""
    if steps < 0 or diag_every < 1:
        raise L.InvalidParameter("evolve: steps >= 0 and diag_every >= 1 required")
    lib = L.lib()
    h = scheme.handle
    be = state.formulation == Formulation.BE
    scheme.load(state)

    def emit(s):
        en, gr, t = C.c_double(), C.c_double(0.0), C.c_double()
        L.check(lib.sfeec_dev_energy(h, C.byref(en)))
        if be:
            L.check(lib.sfeec_dev_gauss_residual(h, C.byref(gr)))
        L.check(lib.sfeec_dev_get_state(h, None, None, C.byref(t)))
        return _row(s, t.value, en.value, gr.value)

    rows = ["step,time,energy,gauss_residual\n", emit(0)]
    s = 0
    while s < steps:
        nxt = min(steps, (s // diag_every + 1) * diag_every)
        L.check(lib.sfeec_dev_advance(h, nxt - s))
        s = nxt
        rows.append(emit(s))
    text = "".join(rows)
    if out:
        with open(out, "w", newline="") as f:
            f.write(text)
    return text


def read_history(text: str) -> np.ndarray:
    """CSV history -> structured array (step, time, energy, gauss_residual)."""
    lines = text.strip().splitlines()
    if not lines or lines[0] != "step,time,energy,gauss_residual":
        raise ValueError("not an evolve history")
    data = [tuple(float(x) for x in ln.split(",")) for ln in lines[1:]]
    arr = np.array(data, dtype=np.float64).reshape(-1, 4)
    return arr


def save_checkpoint(path: str, state: FieldState) -> None:
    np.savez(path, formulation=int(state.formulation), first=state.first, e=state.e,
             time=np.float64(state.time))


def load_checkpoint(path: str) -> FieldState:
    with np.load(path) as z:
        return make_state(Formulation(int(z["formulation"])), z["first"], z["e"],
                          float(z["time"]))
