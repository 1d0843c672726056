#!/usr/bin/env python
"""Exact (rational) reference-element tables of the second-order trimmed
family P2^- Lambda^k on a tetrahedron (BASELINE config 4), written to
paper_2301_01753_b200/csrc/p2_tables.hpp.

The reference implements P2^- only on triangles (form_space.cpp:41-166); the
3-D element here follows the same conventions:

  reference tet s in {s_i >= 0, sum s_i <= 1}, vertices v0 = 0, v1..v3 = e_i,
  barycentrics l0 = 1 - s1 - s2 - s3, l_k = s_k; local vertex order =
  ascending global vertex id, so every sub-simplex is oriented by its
  ascending vertex order.

  1-form DOFs (20): per edge (a,b) (local order 01 02 03 12 13 23) the
    moments of the tangential trace against 1 and 2t-1 along x = v_a +
    t (v_b - v_a)   [form_space.cpp:423, the 2-D edge moments];
    per face (a,b,c) (local order 123 023 013 012), with y = v_a + p (v_b -
    v_a) + q (v_c - v_a), the moments int dp ^ u and int dq ^ u
    [form_space.cpp:131-138, the 2-D interior moments].
  2-form DOFs (15): per face the flux moments against the face
    barycentrics (1-p-q, p, q) [form_space.cpp:141-156]; then the three
    interior moments int dl_k ^ w, k = 1..3.
  3-form DOFs (4): moments against l_0..l_3.

Spanning sets: l_m * Whitney forms (P_2^- = span{l^alpha phi_sigma}); the
dual basis is solved exactly with Fractions, so every table entry is the
correctly rounded double of a rational number.

Proxies: a 1-form u = sum u_k ds_k <-> vector u; a 2-form <-> vector w with
w_1 ds2^ds3 + w_2 ds3^ds1 + w_3 ds1^ds2 (wedge of 1-forms = cross product);
a 3-form <-> scalar rho ds1^ds2^ds3. On a physical tet x = x0 + J s:
  M1_ij = int u_i^T G1 u_j ds, G1 = |det J| J^-1 J^-T
  M2_ij = int w_i^T G2 w_j ds, G2 = J^T J / |det J|
Tables: I1[i][j][k][l] = int u_ik u_jl ds, I2 likewise, C[i][j] =
DOF2_i(d u_j), D[i][j] = DOF3_i(d w_j).
"""
from __future__ import annotations

import os
import sys
from fractions import Fraction as F
from itertools import combinations
from math import factorial

# ---- polynomials in (s1, s2, s3): dict {(a, b, c): Fraction} ---------------


def padd(p, q, cq=F(1)):
    r = dict(p)
    for k, v in q.items():
        r[k] = r.get(k, F(0)) + cq * v
        if r[k] == 0:
            del r[k]
    return r


def pmul(p, q):
    r = {}
    for (a, b, c), u in p.items():
        for (d, e, f), v in q.items():
            k = (a + d, b + e, c + f)
            r[k] = r.get(k, F(0)) + u * v
            if r[k] == 0:
                del r[k]
    return r


def pscale(p, c):
    return {k: v * c for k, v in p.items() if v * c != 0}


def pderiv(p, i):
    r = {}
    for k, v in p.items():
        if k[i] == 0:
            continue
        kk = list(k)
        kk[i] -= 1
        r[tuple(kk)] = r.get(tuple(kk), F(0)) + v * k[i]
    return {k: v for k, v in r.items() if v != 0}


ONE = {(0, 0, 0): F(1)}
S = [{(1, 0, 0): F(1)}, {(0, 1, 0): F(1)}, {(0, 0, 1): F(1)}]
LAM = [padd(padd(padd(ONE, S[0], F(-1)), S[1], F(-1)), S[2], F(-1)), S[0], S[1], S[2]]
DLAM = [(F(-1), F(-1), F(-1)), (F(1), F(0), F(0)), (F(0), F(1), F(0)), (F(0), F(0), F(1))]
VERT = [(F(0), F(0), F(0)), (F(1), F(0), F(0)), (F(0), F(1), F(0)), (F(0), F(0), F(1))]
EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
FACES = [(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)]


def cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def sub(a, b):
    return tuple(x - y for x, y in zip(a, b))


def int_tet(p):
    """int over the reference tet of p."""
    return sum(v * F(factorial(a) * factorial(b) * factorial(c), factorial(a + b + c + 3))
               for (a, b, c), v in p.items())


def subst(p, base, dirs):
    """p(base + sum_m t_m dirs[m]) as a polynomial in the t's (dict over
    exponent tuples of len(dirs))."""
    nd = len(dirs)
    # affine images of s1, s2, s3 in the t variables
    aff = []
    for i in range(3):
        q = {(0,) * nd: base[i]} if base[i] != 0 else {}
        for m in range(nd):
            if dirs[m][i] != 0:
                k = tuple(1 if mm == m else 0 for mm in range(nd))
                q[k] = q.get(k, F(0)) + dirs[m][i]
        aff.append(q)

    def mul(x, y):
        r = {}
        for ka, u in x.items():
            for kb, v in y.items():
                k = tuple(i + j for i, j in zip(ka, kb))
                r[k] = r.get(k, F(0)) + u * v
        return {k: v for k, v in r.items() if v != 0}

    out = {}
    for (a, b, c), v in p.items():
        term = {(0,) * nd: v}
        for i, e in enumerate((a, b, c)):
            for _ in range(e):
                term = mul(term, aff[i])
        for k, w in term.items():
            out[k] = out.get(k, F(0)) + w
    return {k: v for k, v in out.items() if v != 0}


def int_seg(p):  # p over (t,), t in [0, 1]
    return sum(v * F(1, k[0] + 1) for k, v in p.items())


def int_tri(p):  # p over (p, q) on the reference triangle
    return sum(v * F(factorial(a) * factorial(b), factorial(a + b + 2)) for (a, b), v in p.items())


# ---- forms ------------------------------------------------------------------


def whitney1(i, j):
    return tuple(padd(pscale(LAM[i], DLAM[j][k]), pscale(LAM[j], DLAM[i][k]), F(-1))
                 for k in range(3))


def whitney2(i, j, k):
    a, b, c = cross(DLAM[j], DLAM[k]), cross(DLAM[i], DLAM[k]), cross(DLAM[i], DLAM[j])
    out = []
    for m in range(3):
        p = padd(padd(pscale(LAM[i], 2 * a[m]), pscale(LAM[j], -2 * b[m])), pscale(LAM[k], 2 * c[m]))
        out.append(p)
    return tuple(out)


def vec_dot_poly(vec, const):  # sum_k vec[k] * const[k]
    r = {}
    for k in range(3):
        r = padd(r, pscale(vec[k], const[k]))
    return r


def curl(u):
    d = lambda f, i: pderiv(f, i)  # noqa: E731
    return (padd(d(u[2], 1), d(u[1], 2), F(-1)), padd(d(u[0], 2), d(u[2], 0), F(-1)),
            padd(d(u[1], 0), d(u[0], 1), F(-1)))


def div(w):
    return padd(padd(pderiv(w[0], 0), pderiv(w[1], 1)), pderiv(w[2], 2))


def dofs1(u):
    out = []
    for a, b in EDGES:
        t = sub(VERT[b], VERT[a])
        tang = subst(vec_dot_poly(u, t), VERT[a], [t])
        out.append(int_seg(tang))
        out.append(int_seg(pmul_t(tang, {(1,): F(2), (0,): F(-1)})))
    for a, b, c in FACES:
        e1, e2 = sub(VERT[b], VERT[a]), sub(VERT[c], VERT[a])
        up = subst(vec_dot_poly(u, e1), VERT[a], [e1, e2])
        uq = subst(vec_dot_poly(u, e2), VERT[a], [e1, e2])
        out.append(int_tri(uq))                       # int dp ^ u
        out.append(-int_tri(up))                      # int dq ^ u
    return out


def pmul_t(x, y):
    r = {}
    for ka, u in x.items():
        for kb, v in y.items():
            k = tuple(i + j for i, j in zip(ka, kb))
            r[k] = r.get(k, F(0)) + u * v
    return {k: v for k, v in r.items() if v != 0}


def dofs2(w):
    out = []
    for a, b, c in FACES:
        e1, e2 = sub(VERT[b], VERT[a]), sub(VERT[c], VERT[a])
        flux = subst(vec_dot_poly(w, cross(e1, e2)), VERT[a], [e1, e2])
        for lam in ({(0, 0): F(1), (1, 0): F(-1), (0, 1): F(-1)}, {(1, 0): F(1)}, {(0, 1): F(1)}):
            out.append(int_tri(pmul_t(flux, lam)))
    for k in range(3):
        out.append(int_tet(w[k]))                     # int ds_k ^ w = int w_k
    return out


def dofs3(rho):
    return [int_tet(pmul(LAM[m], rho)) for m in range(4)]


def solve_dual(span, dof_fn, dim, combine):
    """Basis dual to dof_fn inside span (exact)."""
    V = [dof_fn(s) for s in span]                     # V[j] = dofs of spanning form j
    # choose dim independent spanning forms (exact elimination on columns)
    chosen, rows = [], []
    for j, col in enumerate(V):
        vec = list(col)
        for (piv, r) in rows:
            if vec[piv] != 0:
                f = vec[piv] / r[piv]
                vec = [x - f * y for x, y in zip(vec, r)]
        nz = [i for i, x in enumerate(vec) if x != 0]
        if nz:
            rows.append((nz[0], vec))
            chosen.append(j)
        if len(chosen) == dim:
            break
    assert len(chosen) == dim, "spanning set does not reach the element dimension"
    # A = V_sub^T (dofs x chosen); basis_i = sum_m B[i][m] span[chosen[m]] with A B^T = I
    A = [[V[chosen[m]][i] for m in range(dim)] for i in range(dim)]
    inv = inverse(A)                                  # A^-1
    basis = []
    for i in range(dim):  # basis_i = sum_m inv[m][i] span[chosen[m]]
        basis.append(combine([(inv[m][i], span[chosen[m]]) for m in range(dim)]))
    return basis


def inverse(A):
    n = len(A)
    M = [list(r) + [F(int(i == j)) for j in range(n)] for i, r in enumerate(A)]
    for c in range(n):
        p = next(r for r in range(c, n) if M[r][c] != 0)
        M[c], M[p] = M[p], M[c]
        pv = M[c][c]
        M[c] = [x / pv for x in M[c]]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c]
                M[r] = [x - f * y for x, y in zip(M[r], M[c])]
    return [r[n:] for r in M]


def comb_vec(terms):
    out = [{}, {}, {}]
    for c, f in terms:
        for k in range(3):
            out[k] = padd(out[k], f[k], c)
    return tuple(out)


def comb_scalar(terms):
    out = {}
    for c, f in terms:
        out = padd(out, f, c)
    return out


def build():
    span1 = [tuple(pmul(LAM[m], f) for f in whitney1(i, j)) for (i, j) in EDGES for m in range(4)]
    span2 = [tuple(pmul(LAM[m], f) for f in whitney2(*t)) for t in combinations(range(4), 3)
             for m in range(4)]
    span3 = [LAM[m] for m in range(4)]
    b1 = solve_dual(span1, dofs1, 20, comb_vec)
    b2 = solve_dual(span2, dofs2, 15, comb_vec)
    b3 = solve_dual(span3, dofs3, 4, comb_scalar)
    # checks: duality
    for basis, fn in ((b1, dofs1), (b2, dofs2), (b3, dofs3)):
        for i, f in enumerate(basis):
            d = fn(f)
            assert all(d[j] == (1 if i == j else 0) for j in range(len(basis)))
    C = [[dofs2(curl(u))[i] for u in b1] for i in range(15)]
    D = [[dofs3(div(w))[i] for w in b2] for i in range(4)]
    I1 = [[[[int_tet(pmul(b1[i][k], b1[j][l])) for l in range(3)] for k in range(3)]
           for j in range(20)] for i in range(20)]
    I2 = [[[[int_tet(pmul(b2[i][k], b2[j][l])) for l in range(3)] for k in range(3)]
           for j in range(15)] for i in range(15)]
    # D C = 0 exactly
    for i in range(4):
        for j in range(20):
            assert sum(D[i][m] * C[m][j] for m in range(15)) == 0
    return dict(C=C, D=D, I1=I1, I2=I2, b1=b1, b2=b2, b3=b3)


def fmt(x: F) -> str:
    v = float(x)
    return repr(v) if v != 0 else "0.0"


def write_header(t, path):
    lines = ["// Generated by tools/gen_p2_tables.py -- exact rational tables of the",
             "// P2^- Lambda^k reference tetrahedron, correctly rounded (DESIGN.md 3.3).",
             "#pragma once", "", "namespace sfeec_b200 {", "namespace p2t {", ""]

    def arr(name, dims, flat):
        lines.append(f"inline constexpr double {name}" + "".join(f"[{d}]" for d in dims) + " = {")
        per = 6
        for i in range(0, len(flat), per):
            lines.append("    " + ", ".join(fmt(x) for x in flat[i:i + per]) + ",")
        lines.append("};")
        lines.append("")

    arr("kC", (15, 20), [x for r in t["C"] for x in r])
    arr("kD", (4, 15), [x for r in t["D"] for x in r])
    arr("kI1", (20, 20, 3, 3), [t["I1"][i][j][k][l] for i in range(20) for j in range(20)
                               for k in range(3) for l in range(3)])
    arr("kI2", (15, 15, 3, 3), [t["I2"][i][j][k][l] for i in range(15) for j in range(15)
                               for k in range(3) for l in range(3)])
    lines += ["}  // namespace p2t", "}  // namespace sfeec_b200", ""]
    with open(path, "w") as f:
        f.write("\n".join(lines))


if __name__ == "__main__":
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
        root, "paper_2301_01753_b200", "csrc", "p2_tables.hpp")
    write_header(build(), out)
    print("wrote", out)
