"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the second-order P2^-
system on the Kuhn tet mesh (BASELINE config 4).

Parity status: **unpinned by the reference** -- its P2^- family is 2-D only
(form_space.cpp:41-166); the 3-D element follows the same DOF conventions
(edge moments against 1 and 2t-1, form_space.cpp:423; face moments int dl_k ^ u,
form_space.cpp:131-138; 2-form moments against barycentrics,
form_space.cpp:141-156), written out in DESIGN.md 3.3. This restatement is
independent of the product's exact-rational tables (tools/gen_p2_tables.py):
it builds the dual basis numerically (Gauss quadrature + pseudo-inverse of
the DOF matrix of the spanning set l_m * Whitney forms), so agreement checks
both derivations. Assembly follows the product's row conventions (ascending
tets, sums from 0.0, exact zeros dropped) for small meshes.
"""
from __future__ import annotations

from itertools import combinations

import numpy as np

from .tetmesh_oracle import LE, LF, OracleTetMesh

GRAD = np.array([[-1.0, -1.0, -1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
VERT = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])


def _lam(s):
    s = np.atleast_2d(s)
    return np.concatenate([1.0 - s.sum(axis=1, keepdims=True), s], axis=1)  # (npts, 4)


# ---- quadrature -----------------------------------------------------------
def gauss_segment(q=4):
    x, w = np.polynomial.legendre.leggauss(q)
    return 0.5 * (x + 1.0), 0.5 * w


def gauss_triangle(q=5):
    """Collapsed (Duffy) Gauss rule on {p, q >= 0, p + q <= 1}."""
    x, w = gauss_segment(q)
    P, W = [], []
    for xi, wi in zip(x, w):
        for yj, wj in zip(x, w):
            P.append((xi, (1.0 - xi) * yj))
            W.append(wi * wj * (1.0 - xi))
    return np.array(P), np.array(W)


def gauss_tet(q=5):
    x, w = gauss_segment(q)
    P, W = [], []
    for a, wa in zip(x, w):
        for b, wb in zip(x, w):
            for c, wc in zip(x, w):
                s1 = a
                s2 = (1.0 - a) * b
                s3 = (1.0 - a) * (1.0 - b) * c
                P.append((s1, s2, s3))
                W.append(wa * wb * wc * (1.0 - a) ** 2 * (1.0 - b))
    return np.array(P), np.array(W)


# ---- spanning forms (vector proxies), their d, evaluated at points ---------
def span1(s):
    """(24, npts, 3) values and (24, npts, 3) curls of l_m phi_ij."""
    lam = _lam(s)
    vals, curls = [], []
    for i, j in LE:
        phi = lam[:, i:i + 1] * GRAD[j] - lam[:, j:j + 1] * GRAD[i]
        cphi = 2.0 * np.cross(GRAD[i], GRAD[j])
        for m in range(4):
            vals.append(lam[:, m:m + 1] * phi)
            curls.append(np.cross(GRAD[m], phi) + lam[:, m:m + 1] * cphi)
    return np.array(vals), np.array(curls)


def span2(s):
    """(16, npts, 3) values and (16, npts) divergences of l_m phi_ijk."""
    lam = _lam(s)
    vals, divs = [], []
    for i, j, k in combinations(range(4), 3):
        phi = 2.0 * (lam[:, i:i + 1] * np.cross(GRAD[j], GRAD[k])
                     - lam[:, j:j + 1] * np.cross(GRAD[i], GRAD[k])
                     + lam[:, k:k + 1] * np.cross(GRAD[i], GRAD[j]))
        dphi = 6.0 * GRAD[i] @ np.cross(GRAD[j], GRAD[k])
        for m in range(4):
            vals.append(lam[:, m:m + 1] * phi)
            divs.append(phi @ GRAD[m] + lam[:, m] * dphi)
    return np.array(vals), np.array(divs)


def span3(s):
    return _lam(s).T.copy()  # (4, npts)


# ---- DOF functionals applied to families of fields -------------------------
def dofs1(field):
    """field(s) -> (nf, npts, 3); returns (nf, 20)."""
    out = []
    t, wt = gauss_segment()
    for a, b in LE:
        tau = VERT[b] - VERT[a]
        pts = VERT[a] + t[:, None] * tau
        tang = field(pts) @ tau                    # (nf, nq)
        out.append(tang @ wt)
        out.append(tang @ (wt * (2.0 * t - 1.0)))
    P, W = gauss_triangle()
    for a, b, c in LF:
        e1, e2 = VERT[b] - VERT[a], VERT[c] - VERT[a]
        pts = VERT[a] + P[:, :1] * e1 + P[:, 1:] * e2
        f = field(pts)
        out.append((f @ e2) @ W)                   # int dp ^ u = int u_q
        out.append(-(f @ e1) @ W)                  # int dq ^ u = -int u_p
    return np.stack(out, axis=1)


def dofs2(field):
    out = []
    P, W = gauss_triangle()
    for a, b, c in LF:
        e1, e2 = VERT[b] - VERT[a], VERT[c] - VERT[a]
        pts = VERT[a] + P[:, :1] * e1 + P[:, 1:] * e2
        flux = field(pts) @ np.cross(e1, e2)
        for lam in (1.0 - P[:, 0] - P[:, 1], P[:, 0], P[:, 1]):
            out.append(flux @ (W * lam))
    Pt, Wt = gauss_tet()
    f = field(Pt)
    for k in range(3):
        out.append(f[:, :, k] @ Wt)
    return np.stack(out, axis=1)


def dofs3(field):
    Pt, Wt = gauss_tet()
    lam = _lam(Pt)
    f = field(Pt)
    return np.stack([f @ (Wt * lam[:, m]) for m in range(4)], axis=1)


class P2Element:
    """Dual bases and element tables of P2^- on the reference tet."""

    def __init__(self):
        V1 = dofs1(lambda s: span1(s)[0])          # (24, 20)
        V2 = dofs2(lambda s: span2(s)[0])          # (16, 15)
        V3 = dofs3(span3)                          # (4, 4)
        # basis_i = sum_j A[i, j] span_j with A V = I (minimum-norm right inverse)
        self.A1 = np.linalg.pinv(V1)               # (20, 24)
        self.A2 = np.linalg.pinv(V2)               # (15, 16)
        self.A3 = np.linalg.inv(V3)
        for A, V in ((self.A1, V1), (self.A2, V2), (self.A3, V3)):
            assert np.allclose(A @ V, np.eye(A.shape[0]), atol=1e-12)

    def basis1(self, s):
        v, c = span1(s)
        return np.einsum("ij,jpk->ipk", self.A1, v), np.einsum("ij,jpk->ipk", self.A1, c)

    def basis2(self, s):
        v, d = span2(s)
        return np.einsum("ij,jpk->ipk", self.A2, v), self.A2 @ d

    def tables(self):
        C = dofs2(lambda s: self.basis1(s)[1]).T                  # (15, 20)
        D = dofs3(lambda s: self.basis2(s)[1]).T                  # (4, 15)
        Pt, Wt = gauss_tet()
        u, _ = self.basis1(Pt)
        w, _ = self.basis2(Pt)
        I1 = np.einsum("ipk,jpl,p->ijkl", u, u, Wt)
        I2 = np.einsum("ipk,jpl,p->ijkl", w, w, Wt)
        return dict(C=C, D=D, I1=I1, I2=I2)


# ---- numbering and assembly on the oracle mesh ------------------------------
class OracleP2:
    def __init__(self, mesh: OracleTetMesh, element: P2Element | None = None):
        self.m = m = mesh
        self.el = element or P2Element()
        self.tab = self.el.tables()
        n, N = m.n, m.n + 1
        from .tetmesh_oracle import ET, FT
        ne, nf, nt = len(m.edge_vertices), len(m.face_vertices), len(m.tet_vertices)
        e1 = -np.ones((ne, 2), np.int64)
        f1 = -np.ones((nf, 2), np.int64)
        f2 = -np.ones((nf, 3), np.int64)
        t2 = -np.ones((nt, 3), np.int64)
        a1 = a2 = 0
        for k in range(N):
            for j in range(N):
                for ib in range(0, N, 32):
                    ie = min(ib + 32, N)
                    for t in range(7):
                        for s in range(2):
                            for i in range(ib, ie):
                                e = m.eid[m.vid(i, j, k), t]
                                if e >= 0:
                                    e1[e, s] = a1
                                    a1 += 1
                    for f, (ta, tb) in enumerate(FT):
                        for s in range(2):
                            for i in range(ib, ie):
                                fi = m.fid[m.vid(i, j, k), f]
                                c = (i, j, k)
                                bnd = any(ET[ta][d] == 0 and ET[tb][d] == 0 and c[d] in (0, n)
                                          for d in range(3))
                                if fi >= 0 and not bnd:
                                    f1[fi, s] = a1
                                    a1 += 1
                    for f in range(12):
                        for s in range(3):
                            for i in range(ib, ie):
                                fi = m.fid[m.vid(i, j, k), f]
                                if fi >= 0:
                                    f2[fi, s] = a2
                                    a2 += 1
                    if j < n and k < n:
                        for p in range(6):
                            for s in range(3):
                                for i in range(ib, min(ie, n)):
                                    cube = i + n * (j + n * k)
                                    t2[6 * cube + p, s] = a2
                                    a2 += 1
        self.e1, self.f1, self.f2, self.t2 = e1, f1, f2, t2
        self.n1, self.n2, self.n3 = a1, a2, 4 * nt
        self.local = []
        for t, v in enumerate(m.tet_vertices):
            d1, d2 = [], []
            for a, b in LE:
                e = m.edge(v[a], v[b])
                d1 += [e1[e, 0], e1[e, 1]] if e >= 0 else [-1, -1]
            for q in LF:
                fi = m.face(*(v[list(q)]))
                d1 += [f1[fi, 0], f1[fi, 1]]
                d2 += list(f2[fi])
            d2 += list(t2[t])
            self.local.append((np.array(d1), np.array(d2)))

    def metric(self, t):
        v = self.m.tet_vertices[t]
        x = self.m.xyz[v]
        J = (x[1:] - x[0]).T
        det = np.linalg.det(J)
        Ji = np.linalg.inv(J)
        return abs(det) * Ji @ Ji.T, J.T @ J / abs(det), det

    def _assemble(self, nrows, ncols, contribs):
        rows = [dict() for _ in range(nrows)]
        for r, c, v in contribs:
            rows[r][c] = rows[r].get(c, 0.0) + v
        return [sorted((c, v) for c, v in row.items() if v != 0.0) for row in rows]

    def curl_rows(self):
        C = self.tab["C"]
        seen, contribs = set(), []
        for t, (d1, d2) in enumerate(self.local):
            for p in range(15):
                if d2[p] in seen:
                    continue  # face rows from their first tet
                seen.add(d2[p])
                for q in range(20):
                    if d1[q] >= 0 and abs(C[p, q]) > 1e-12:
                        contribs.append((d2[p], d1[q], C[p, q]))
        return self._assemble(self.n2, self.n1, contribs)

    def div_rows(self):
        D = self.tab["D"]
        contribs = []
        for t, (_, d2) in enumerate(self.local):
            for p in range(4):
                for q in range(15):
                    if abs(D[p, q]) > 1e-12:
                        contribs.append((4 * t + p, d2[q], D[p, q]))
        return self._assemble(self.n3, self.n2, contribs)

    def mass_rows(self, form):
        I = self.tab["I1" if form == 1 else "I2"]
        contribs = []
        for t, (d1, d2) in enumerate(self.local):
            g1, g2, _ = self.metric(t)
            g = g1 if form == 1 else g2
            dl = d1 if form == 1 else d2
            Me = np.einsum("kl,ijkl->ij", g, I)
            for p in range(len(dl)):
                for q in range(len(dl)):
                    if dl[p] >= 0 and dl[q] >= 0:
                        contribs.append((dl[p], dl[q], Me[p, q]))
        n = self.n1 if form == 1 else self.n2
        return self._assemble(n, n, contribs)
