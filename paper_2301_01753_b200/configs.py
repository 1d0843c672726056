"""BASELINE.json configurations: operators and seeded initial states (setup).

  tet_system(n, jitter, seed)       configs 1/3/5: Kuhn tets, PEC, P1-, SPAI S(M1)
  initial_gaussian(sys, seed)       config 1: A ~ N(0,1) on interior edges, B0 = C A, E0 = 0
  initial_pulse(sys, seed, npulses) configs 3/5: Gaussian pulse(s) of width 0.1 in A
  cfl_dt(scheme)                    dt = 0.5 * dt_CFL, dt_CFL = 2 / (c sqrt(lambda)),
                                    lambda from the reference power iteration
                                    (dynamics.cpp:114-133)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import inputs
from .scheme import SparseOperator, TetMesh, spai_approximate_inverse


@dataclass
class TetSystem:
    mesh: TetMesh
    c: SparseOperator
    m1: SparseOperator
    m2: SparseOperator
    d: SparseOperator
    q: SparseOperator       # SPAI of M1 (not symmetrised; SplitScheme does that)
    spai_report: dict

    @property
    def n1(self):
        return self.c.cols

    @property
    def n2(self):
        return self.c.rows


def tet_system(n: int, jitter: float = 0.1, seed: int = 0, pattern: str = "m1") -> TetSystem:
    mesh = TetMesh(n, jitter, seed)
    c, m1, m2, d = mesh.curl(), mesh.mass1(), mesh.mass2(), mesh.div()
    q, rep = spai_approximate_inverse(m1, pattern)
    return TetSystem(mesh, c, m1, m2, d, q, rep)


def spmv(a: SparseOperator, x: np.ndarray) -> np.ndarray:
    """Host CSR product for setup only (initial B0 = C A)."""
    rows = np.repeat(np.arange(a.rows), np.diff(a.row_ptr))
    y = np.zeros(a.rows)
    np.add.at(y, rows, a.val * x[a.col_idx])
    return y


def initial_gaussian(sys: TetSystem, seed: int = 1):
    a = inputs.gaussian(seed, sys.n1)
    return spmv(sys.c, a), np.zeros(sys.n1), a


def initial_pulse(sys: TetSystem, seed: int = 1, npulses: int = 1, sigma: float = 0.1):
    xyz, ev, _, _ = sys.mesh.geometry()
    a = inputs.pulse_one_form(xyz, ev, seed, sigma, npulses)
    return spmv(sys.c, a), np.zeros(sys.n1), a


def cfl_dt(scheme) -> float:
    """0.5 x the CFL estimate: nu(dt) = dt c sqrt(lambda) and dt_CFL = 2/(c sqrt(lambda))."""
    nu = scheme.cfl_number()
    return 0.5 * 2.0 * scheme.dt() / nu
