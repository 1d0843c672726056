"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference's consistent
Q1- mass matrices on the periodic cubical lattice:

  mass_matrix            proj/src/operators.cpp:133-179 (per-cell quadrature,
                         dot over components from 0, exact symmetric mirror,
                         triplets summed in input order by operator_from_triplets,
                         sparse.cpp:20-61)
  Q1 element             form_space.cpp:295-321 (no transform on cubes,
                         jac_abs = dx dy dz, form_space.cpp:210-211)
  cube rule, order 3     quadrature.cpp:90-107 (2-point Gauss-Legendre per axis)
  local DOF order        mesh_cubical.cpp:136-165
  ids                    axis * N + vid(i, j, k), vid = i + nx (j + ny k)

Pinned against the reference's own golden values (test_operators.cpp:110-149:
4 dV/9, dV/9, dV/36, 0 across components, 2 dV/3, dV/6, row sums dV); the
product's host builder (host_yee.cpp build_yee_mass) must equal it bitwise.
"""
from __future__ import annotations

import numpy as np

_GX = (-0.5773502691896257645, 0.5773502691896257645)
_BB = ((0, 0), (1, 0), (0, 1), (1, 1))


def _rule():
    pts, w = [], []
    for k in range(2):
        for j in range(2):
            for i in range(2):
                pts.append((0.5 * (_GX[i] + 1.0), 0.5 * (_GX[j] + 1.0), 0.5 * (_GX[k] + 1.0)))
                w.append(0.125 * 1.0 * 1.0 * 1.0)
    return pts, w


def _lshape(b, t):
    return t if b else 1.0 - t


def element(form, dx, dy, dz):
    pts, w = _rule()
    nl = 12 if form == 1 else 6
    ref = []
    for r in pts:
        vals = [[0.0, 0.0, 0.0] for _ in range(nl)]
        l = 0
        for a in range(3):
            a1, a2 = (a + 1) % 3, (a + 2) % 3
            if form == 1:
                for b1, b2 in _BB:
                    vals[l][a] = _lshape(b1, r[a1]) * _lshape(b2, r[a2])
                    l += 1
            else:
                for b in (0, 1):
                    vals[l][a] = _lshape(b, r[a])
                    l += 1
        ref.append(vals)
    scale = dx * dy * dz
    me = [[0.0] * nl for _ in range(nl)]
    for i in range(nl):
        for j in range(i, nl):
            acc = 0.0
            for q in range(len(pts)):
                dot = 0.0
                for k in range(3):
                    dot += ref[q][i][k] * ref[q][j][k]
                acc += w[q] * dot
            acc *= scale
            me[i][j] = me[j][i] = acc
    return me


def mass_periodic(nx, ny, nz, dx, dy, dz, form):
    """Rows (sorted (col, val) lists) of the periodic-lattice M1 / M2."""
    N = nx * ny * nz
    vid = lambda i, j, k: (i % nx) + nx * ((j % ny) + ny * (k % nz))  # noqa: E731
    me = element(form, dx, dy, dz)
    trip = []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                c = (i, j, k)
                dofs = []
                for a in range(3):
                    a1, a2 = (a + 1) % 3, (a + 2) % 3
                    if form == 1:
                        for b1, b2 in _BB:
                            p = list(c)
                            p[a1] += b1
                            p[a2] += b2
                            dofs.append(a * N + vid(*p))
                    else:
                        for b in (0, 1):
                            p = list(c)
                            p[a] += b
                            dofs.append(a * N + vid(*p))
                nl = len(dofs)
                for x in range(nl):
                    for y in range(nl):
                        trip.append((dofs[x], dofs[y], me[x][y]))
    rows = [dict() for _ in range(3 * N)]
    for r, c, v in trip:  # input order within each (r, c): cell, then slot
        rows[r][c] = rows[r].get(c, 0.0) + v
    return [sorted((c, v) for c, v in row.items() if v != 0.0) for row in rows]
