"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the 3-D construction.

Parity status: **unpinned by the reference** -- the reference has no 3-D tet
meshes, PEC walls or P1- on tets. This file restates the
construction contract written in DESIGN.md ("Tet mesh, numbering and Whitney
element matrices") independently of the product's C++
(paper_2301_01753_b200/csrc/host_tet.cpp), following the reference's
conventions:
  * ascending-vertex-id orientation (reference SPEC.md:78,
    mesh_simplicial.cpp:16-38);
  * integral DOFs -> d = signed incidence (operators.cpp:29-42, P1 branch);
  * element matrices with an exact symmetric mirror, duplicates summed in
    ascending cell order from 0.0, exact zeros dropped (operators.cpp:133-179,
    sparse.cpp:20-61);
  * make_pattern S(M1) / S(M1^2) (spai.cpp:31-72).
The tests check the product against it bit for bit (connectivity, signs,
patterns, mass values) and pin both against the invariants the reference's
own tests assert. SPAI values are checked against a
numpy least-squares solve with a tolerance (the reference solves with Eigen
LDLT, which is absent here).
"""
from __future__ import annotations

import itertools

import numpy as np

ET = np.array([(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (0, 1, 1), (1, 0, 1), (1, 1, 1)])
FT = [(0, 3), (1, 3), (1, 4), (2, 4), (0, 5), (2, 5), (0, 6), (1, 6), (2, 6), (3, 6), (4, 6), (5, 6)]
PERM = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
LE = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
LF = [(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)]
BLOCK = 32


def _u01(seed, k):
    k = np.asarray(k, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (k + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


class OracleTetMesh:
    def __init__(self, n, jitter=0.1, seed=0):
        self.n = n
        N = n + 1
        self.nv = N ** 3
        vid = np.arange(self.nv)
        c = np.stack([vid % N, (vid // N) % N, vid // (N * N)], axis=1)
        self.coords = c
        h = 1.0 / n
        interior = np.all((c > 0) & (c < n), axis=1)
        xyz = c.astype(np.float64) * h
        if jitter > 0:
            for d in range(3):
                u = _u01(seed, 3 * vid + d)
                jit = xyz[:, d] + (jitter * h) * (2.0 * u - 1.0)
                xyz[:, d] = np.where(interior, jit, xyz[:, d])
        self.xyz = xyz
        # numbering loops (k, j, x-block, type, i) -- explicit Python loops
        eid = -np.ones((self.nv, 7), np.int64)
        fid = -np.ones((self.nv, 12), np.int64)
        ne = nf = 0
        ev, fv = [], []
        for k in range(N):
            for j in range(N):
                for ib in range(0, N, BLOCK):
                    ie = min(ib + BLOCK, N)
                    for t in range(7):
                        for i in range(ib, ie):
                            e = (i + ET[t][0], j + ET[t][1], k + ET[t][2])
                            if max(e) > n:
                                continue
                            cc = (i, j, k)
                            if any(ET[t][d] == 0 and cc[d] in (0, n) for d in range(3)):
                                continue
                            eid[self.vid(i, j, k), t] = ne
                            ev.append((self.vid(i, j, k), self.vid(*e)))
                            ne += 1
                    for f, (t1, t2) in enumerate(FT):
                        for i in range(ib, ie):
                            e2 = (i + ET[t2][0], j + ET[t2][1], k + ET[t2][2])
                            if max(e2) > n:
                                continue
                            e1 = (i + ET[t1][0], j + ET[t1][1], k + ET[t1][2])
                            fid[self.vid(i, j, k), f] = nf
                            fv.append((self.vid(i, j, k), self.vid(*e1), self.vid(*e2)))
                            nf += 1
        self.eid, self.fid = eid, fid
        self.edge_vertices = np.array(ev, np.int64).reshape(-1, 2)
        self.face_vertices = np.array(fv, np.int64).reshape(-1, 3)
        tv = []
        for kc in range(n):
            for jc in range(n):
                for ic in range(n):
                    for p in PERM:
                        cc = [ic, jc, kc]
                        vs = [self.vid(*cc)]
                        for a in p:
                            cc[a] += 1
                            vs.append(self.vid(*cc))
                        tv.append(vs)
        self.tet_vertices = np.array(tv, np.int64).reshape(-1, 4)
        self._edge_lookup = {tuple(e): i for i, e in enumerate(self.edge_vertices)}
        self._face_lookup = {tuple(f): i for i, f in enumerate(self.face_vertices)}

    def vid(self, i, j, k):
        N = self.n + 1
        return i + N * (j + N * k)

    def edge(self, a, b):
        return self._edge_lookup.get((a, b), -1)

    def face(self, a, b, c):
        return self._face_lookup[(a, b, c)]

    # ---- incidence ------------------------------------------------------
    def curl_rows(self):
        rows = []
        for v0, v1, v2 in self.face_vertices:
            r = {}
            for (a, b), s in (((v1, v2), 1.0), ((v0, v2), -1.0), ((v0, v1), 1.0)):
                e = self.edge(a, b)
                if e >= 0:
                    r[e] = r.get(e, 0.0) + s
            rows.append(sorted((c, v) for c, v in r.items() if v != 0.0))
        return rows

    def div_rows(self):
        rows = []
        for v in self.tet_vertices:
            r = {}
            for f, s in zip(LF, (1.0, -1.0, 1.0, -1.0)):
                r[self.face(*(v[list(f)]))] = s
            rows.append(sorted(r.items()))
        return rows

    # ---- Whitney element matrices (vectorised over tets, same op order) --
    def elements(self):
        x = self.xyz[self.tet_vertices]  # T x 4 x 3
        e = x[:, 1:, :] - x[:, :1, :]
        def cross(u, v):
            return np.stack([u[:, 1] * v[:, 2] - u[:, 2] * v[:, 1],
                             u[:, 2] * v[:, 0] - u[:, 0] * v[:, 2],
                             u[:, 0] * v[:, 1] - u[:, 1] * v[:, 0]], axis=1)
        c12, c20, c01 = cross(e[:, 1], e[:, 2]), cross(e[:, 2], e[:, 0]), cross(e[:, 0], e[:, 1])
        vol6 = e[:, 0, 0] * c12[:, 0] + e[:, 0, 1] * c12[:, 1] + e[:, 0, 2] * c12[:, 2]
        gl = np.zeros((len(x), 4, 3))
        gl[:, 1] = c12 / vol6[:, None]
        gl[:, 2] = c20 / vol6[:, None]
        gl[:, 3] = c01 / vol6[:, None]
        gl[:, 0] = -((gl[:, 1] + gl[:, 2]) + gl[:, 3])
        vol = np.abs(vol6) / 6.0
        ml = np.zeros((len(x), 4, 4))
        g = np.zeros((len(x), 4, 4))
        for a in range(4):
            for b in range(4):
                ml[:, a, b] = vol / 10.0 if a == b else vol / 20.0
                g[:, a, b] = (gl[:, a, 0] * gl[:, b, 0] + gl[:, a, 1] * gl[:, b, 1]) + gl[:, a, 2] * gl[:, b, 2]
        m1 = np.zeros((len(x), 6, 6))
        for p in range(6):
            for q in range(p, 6):
                i, j = LE[p]
                k, l = LE[q]
                v = ml[:, i, k] * g[:, j, l]
                v = v - ml[:, i, l] * g[:, j, k]
                v = v - ml[:, j, k] * g[:, i, l]
                v = v + ml[:, j, l] * g[:, i, k]
                m1[:, p, q] = v
                m1[:, q, p] = v
        cv = np.zeros((len(x), 4, 3, 3))
        ci = np.zeros((4, 3), int)
        for f, (a, b, c) in enumerate(LF):
            for t, (p0, p1, p2) in enumerate(((a, b, c), (b, c, a), (c, a, b))):
                ci[f, t] = p0
                cv[:, f, t] = cross(gl[:, p1], gl[:, p2])
        m2 = np.zeros((len(x), 4, 4))
        for f in range(4):
            for h in range(f, 4):
                acc = np.zeros(len(x))
                for s in range(3):
                    for t in range(3):
                        dot = (cv[:, f, s, 0] * cv[:, h, t, 0] + cv[:, f, s, 1] * cv[:, h, t, 1]) \
                            + cv[:, f, s, 2] * cv[:, h, t, 2]
                        acc = acc + ml[:, ci[f, s], ci[h, t]] * dot
                acc = 4.0 * acc
                m2[:, f, h] = acc
                m2[:, h, f] = acc
        return vol6, m1, m2

    def mass(self, form):
        """Assembled mass (CSR tuple): per (row, col), contributions summed in
        ascending tet order starting from 0.0; exact zeros dropped; also the
        structural nnz (entities sharing a tet)."""
        _, m1, m2 = self.elements()
        loc = m1 if form == 1 else m2
        if form == 1:
            ids = np.array([[self.edge(t[a], t[b]) for a, b in LE] for t in self.tet_vertices])
            n = len(self.edge_vertices)
        else:
            ids = np.array([[self.face(*t[list(f)]) for f in LF] for t in self.tet_vertices])
            n = len(self.face_vertices)
        nl = ids.shape[1]
        T = len(ids)
        r = np.repeat(ids, nl, axis=1).reshape(T, nl, nl)
        c = np.tile(ids, (1, nl)).reshape(T, nl, nl)
        t = np.broadcast_to(np.arange(T)[:, None, None], (T, nl, nl))
        keep = (r >= 0) & (c >= 0)
        r, c, t, v = r[keep], c[keep], t[keep], loc[keep]
        order = np.lexsort((t, c, r))
        r, c, v = r[order], c[order], v[order]
        key = r * n + c
        starts = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
        counts = np.diff(np.r_[starts, len(key)])
        acc = np.zeros(len(starts))
        for rank in range(counts.max()):
            sel = counts > rank
            acc[sel] = acc[sel] + v[starts[sel] + rank]
        rr, cc = r[starts], c[starts]
        structural = len(starts)
        nz = acc != 0.0
        rr, cc, acc = rr[nz], cc[nz], acc[nz]
        rp = np.zeros(n + 1, np.int64)
        np.add.at(rp, rr + 1, 1)
        rp = np.cumsum(rp)
        return (n, n, rp, cc.astype(np.int32), acc), structural


def pattern(m, kind):
    """make_pattern, spai.cpp:31-72 (rows of a CSR tuple)."""
    n, _, rp, ci, _ = m
    rows = [ci[rp[i]:rp[i + 1]] for i in range(n)]
    if kind == "diagonal":
        return [np.array([i]) for i in range(n)]
    if kind == "m1":
        return [r.copy() for r in rows]
    return [np.unique(np.concatenate([rows[j] for j in rows[i]])) for i in range(n)]


def spai_lstsq(m, pat):
    """Column-by-column least squares min ||M q - e_l|| over the pattern
    (numpy lstsq on the dense restriction) -- the mathematical definition the
    reference's normal-equation solve implements (spai.cpp:176-233)."""
    n, _, rp, ci, va = m
    dense = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(rp))
    dense[rows, ci] = va
    cols = []
    for l in range(n):
        idx = pat[l]
        e = np.zeros(n)
        e[l] = 1.0
        q, *_ = np.linalg.lstsq(dense[:, idx], e, rcond=None)
        cols.append(q)
    return cols
