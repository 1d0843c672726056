"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the L^2 error of a Whitney
1-form on the Kuhn tet mesh (reference operators.cpp:181-257 l2_error: the
sum over cells of sum_q w_q |w_h(x_q) - f(x_q)|^2 |J|, relative to the same
sum of |f|^2), for the device kernel in paper_2301_01753_b200/csrc/l2_error.cu.

The analytic forms are the PEC cube's TE cavity family: kind 0 A_m =
sin(m pi y) sin(m pi z) dx, kind 1 curl curl A_m = 2 (m pi)^2 A_m. The cell
rule is the collapsed (Duffy) product of 4-point Gauss-Legendre rules; the
canonical projection integrates A_m . t along each edge with 4-point
Gauss-Legendre. Parity: unpinned by the reference (it has no 3-D tets); the
tests pin it by the exactness of the rule and the convergence of the error.
"""
from __future__ import annotations

import numpy as np

from .tetmesh_oracle import LE, OracleTetMesh

_X, _W = np.polynomial.legendre.leggauss(4)
GLX, GLW = (_X + 1.0) / 2.0, _W / 2.0


def analytic(kind, mode, x):
    k = mode * np.pi
    a = np.sin(k * x[..., 1]) * np.sin(k * x[..., 2])
    f = np.zeros(x.shape)
    f[..., 0] = 2.0 * k * k * a if kind == 1 else a
    return f


def project_cavity(mesh: OracleTetMesh, mode: int) -> np.ndarray:
    xa = mesh.xyz[mesh.edge_vertices[:, 0]]
    d = mesh.xyz[mesh.edge_vertices[:, 1]] - xa
    out = np.zeros(len(xa))
    for s, w in zip(GLX, GLW):
        f = analytic(0, mode, xa + s * d)
        out += w * np.sum(f * d, axis=1)
    return out


def tet_rule():
    """(barycentrics [64, 4], weights [64]) on the unit tet (sum 1/6)"""
    lam, wts = [], []
    for i in range(4):
        for j in range(4):
            for k in range(4):
                u, v, s = GLX[i], GLX[j], GLX[k]
                l1, l2, l3 = u, v * (1 - u), s * (1 - u) * (1 - v)
                lam.append((1 - l1 - l2 - l3, l1, l2, l3))
                wts.append(GLW[i] * GLW[j] * GLW[k] * (1 - u) ** 2 * (1 - v))
    return np.array(lam), np.array(wts)


def l2_error(mesh: OracleTetMesh, w: np.ndarray, kind: int, mode: int):
    tv = mesh.tet_vertices
    X = mesh.xyz[tv]  # T x 4 x 3
    e = X[:, 1:] - X[:, :1]
    c12 = np.cross(e[:, 1], e[:, 2])
    c20 = np.cross(e[:, 2], e[:, 0])
    c01 = np.cross(e[:, 0], e[:, 1])
    vol6 = np.einsum("td,td->t", e[:, 0], c12)
    gl = np.zeros((len(tv), 4, 3))
    gl[:, 1], gl[:, 2], gl[:, 3] = c12 / vol6[:, None], c20 / vol6[:, None], c01 / vol6[:, None]
    gl[:, 0] = -(gl[:, 1] + gl[:, 2] + gl[:, 3])
    we = np.zeros((len(tv), 6))
    for q, (a, b) in enumerate(LE):
        ids = np.array([mesh.edge(int(x), int(y)) for x, y in zip(tv[:, a], tv[:, b])])
        we[:, q] = np.where(ids >= 0, w[np.maximum(ids, 0)], 0.0)
    lam, wq = tet_rule()
    err = ex = 0.0
    for p in range(len(wq)):
        x = np.einsum("a,tad->td", lam[p], X)
        disc = np.zeros_like(x)
        for q, (a, b) in enumerate(LE):
            disc += we[:, q, None] * (lam[p, a] * gl[:, b] - lam[p, b] * gl[:, a])
        f = analytic(kind, mode, x)
        err += np.sum(wq[p] * np.sum((disc - f) ** 2, axis=1) * np.abs(vol6))
        ex += np.sum(wq[p] * np.sum(f * f, axis=1) * np.abs(vol6))
    return np.sqrt(err), np.sqrt(err) / np.sqrt(ex)
