"""CPU: the 3-D tet construction (host C++) against the numpy construction
oracle (bitwise) and the invariants the reference's tests assert, restated in
3-D."""
import numpy as np
import pytest
import scipy.linalg as sla

import paper_2301_01753_b200 as S
from oracle import tetmesh_oracle as TO


def tup(a):
    return (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7])
def test_counts_match_appendix_a(n):
    m = S.TetMesh(n, 0.1, 3)
    assert m.n_vertices == (n + 1) ** 3
    assert m.n_edges == 7 * n ** 3 - 9 * n ** 2 + 3 * n
    assert m.n_faces == 12 * n ** 3 + 6 * n ** 2
    assert m.n_tets == 6 * n ** 3
    assert m.curl().nnz() == 36 * n ** 3 - 48 * n ** 2 + 18 * n
    assert m.mass1().nnz() == 115 * n ** 3 - 261 * n ** 2 + 195 * n - 48


@pytest.mark.parametrize("n,jit,seed", [(3, 0.1, 7), (4, 0.15, 11), (2, 0.0, 0)])
def test_construction_bitwise_equals_oracle(n, jit, seed):
    m = S.TetMesh(n, jit, seed)
    o = TO.OracleTetMesh(n, jit, seed)
    xyz, ev, fv, tv = m.geometry()
    assert np.array_equal(xyz, o.xyz)
    assert np.array_equal(ev, o.edge_vertices)
    assert np.array_equal(fv, o.face_vertices)
    assert np.array_equal(tv, o.tet_vertices)
    # orientation: ascending vertex ids
    assert np.all(ev[:, 0] < ev[:, 1]) and np.all(np.diff(fv, axis=1) > 0)
    assert np.all(np.diff(tv, axis=1) > 0)
    for op, rows in ((m.curl(), o.curl_rows()), (m.div(), o.div_rows())):
        for r, want in enumerate(rows):
            got = list(zip(op.row_cols(r).tolist(), op.row_vals(r).tolist()))
            assert got == want, (r, got, want)
    for form, op in ((1, m.mass1()), (2, m.mass2())):
        (rows, cols, rp, ci, va), structural = o.mass(form)
        assert np.array_equal(op.row_ptr, rp) and np.array_equal(op.col_idx, ci)
        assert np.array_equal(op.val, va), f"M{form} values differ"
        if form == 2:
            assert structural == 84 * n ** 3 + 6 * n ** 2


@pytest.mark.parametrize("n", [2, 3])
def test_exact_complex_and_spd(n):
    m = S.TetMesh(n, 0.1, 5)
    c, d = m.curl().to_dense(), m.div().to_dense()
    assert np.all(d @ c == 0.0)  # D C = 0 exactly (test_operators.cpp:43-65)
    for op in (m.mass1(), m.mass2()):
        a = op.to_dense()
        assert np.array_equal(a, a.T)  # exact symmetric mirror
        assert np.linalg.eigvalsh(a).min() > 0  # SPD (test_operators.cpp:173-187)
    # each face has exactly three +-1 boundary entries when all edges are interior
    full = [r for r in range(m.n_faces) if np.diff(m.curl().row_ptr)[r] == 3]
    assert full and all(sorted(m.curl().row_vals(r)) == [-1.0, 1.0, 1.0] for r in full)


def test_mass_couples_only_entities_sharing_a_tet():
    m = S.TetMesh(3, 0.1, 2)
    o = TO.OracleTetMesh(3, 0.1, 2)
    share = set()
    for t in o.tet_vertices:
        es = [o.edge(t[a], t[b]) for a, b in TO.LE]
        es = [e for e in es if e >= 0]
        share.update((a, b) for a in es for b in es)
    m1 = m.mass1()
    for r in range(m1.rows):
        for c in m1.row_cols(r):
            assert (r, int(c)) in share


def test_curl_curl_spectrum_converges_to_cavity_modes():
    """Physics pin of C, M1, M2: the lowest nonzero generalised eigenvalue of
    (C^T M2 C, M1) on the unit PEC cube approximates the TE(1,1,0) cavity
    mode k^2 = 2 pi^2 (triple degenerate); the kernel has dimension equal to
    the number of interior vertices (gradients)."""
    n = 6
    m = S.TetMesh(n, 0.1, 9)
    c, m1, m2 = m.curl().to_dense(), m.mass1().to_dense(), m.mass2().to_dense()
    k = c.T @ m2 @ c
    w = sla.eigh(k, m1, eigvals_only=True)
    kernel = np.sum(w < 1e-8 * w.max())
    assert kernel == (n - 1) ** 3
    lowest = w[kernel:kernel + 3]
    assert np.allclose(lowest, 2 * np.pi ** 2, rtol=0.06), lowest


def test_projected_constant_is_curl_free():
    """C applied to the canonical projection of a constant 1-form vanishes
    (test_operators.cpp:207-221)."""
    m = S.TetMesh(4, 0.1, 1)
    xyz, ev, _, _ = m.geometry()
    u = np.array([0.3, -1.2, 0.7])
    a = (xyz[ev[:, 1]] - xyz[ev[:, 0]]) @ u
    c = m.curl()
    full = np.diff(c.row_ptr) == 3  # faces whose edges are all interior (PEC drops the rest)
    assert full.sum() > 0
    assert np.max(np.abs((c.to_dense() @ a)[full])) <= 1e-14


@pytest.mark.parametrize("kind", ["diagonal", "m1", "m1sq"])
def test_spai_pattern_bitwise_and_values(kind):
    m = S.TetMesh(3, 0.1, 4)
    m1 = m.mass1()
    pat = S.make_pattern(m1, kind)
    want = TO.pattern(tup(m1), kind)
    for r in range(m1.rows):
        assert np.array_equal(pat.row_cols(r), want[r])
    q, rep = S.spai_approximate_inverse(m1, kind)
    assert rep["fallback_columns"] == 0
    cols = TO.spai_lstsq(tup(m1), want)
    qd = q.to_dense()
    for l in range(m1.rows):
        got = qd[want[l], l]
        assert np.allclose(got, cols[l], rtol=1e-9, atol=1e-12 * np.abs(cols[l]).max())
    # reported Frobenius residual equals the direct computation (test_spai.cpp:118-133)
    r = m1.to_dense() @ qd - np.eye(m1.rows)
    assert rep["frobenius_residual"] == pytest.approx(np.linalg.norm(r), rel=1e-6)


def test_spai_residual_monotone_and_diagonal_closed_form():
    m = S.TetMesh(3, 0.1, 4)
    m1 = m.mass1()
    res = [S.spai_approximate_inverse(m1, k)[1]["frobenius_residual"]
           for k in ("diagonal", "m1", "m1sq")]
    assert res[0] >= res[1] >= res[2]  # nested patterns (test_spai.cpp:118-133)
    q, _ = S.spai_approximate_inverse(m1, "diagonal")
    a = m1.to_dense()
    # diagonal SPAI column = M_ll / ||M(:, l)||^2 (test_spai.cpp:97-108)
    want = np.diag(a) / np.sum(a * a, axis=0)
    assert np.allclose(np.diag(q.to_dense()), want, rtol=1e-12)


def test_spai_columns_are_stationary():
    """First-order optimality of every column (test_spai.cpp:135-168):
    M(:, I)^T (M q - e_l) = 0 on the pattern."""
    m = S.TetMesh(2, 0.1, 8)
    m1 = m.mass1()
    q, _ = S.spai_approximate_inverse(m1, "m1")
    a, qd = m1.to_dense(), q.to_dense()
    for l in range(m1.rows):
        idx = m1.row_cols(l)
        r = a @ qd[:, l]
        r[l] -= 1.0
        assert np.max(np.abs(a[:, idx].T @ r)) <= 1e-12


@pytest.mark.parametrize("nzg,k0,k1", [(5, 1, 5), (5, 0, 3), (6, 2, 5)])
def test_slab_rows_equal_whole_mesh_rows(nzg, k0, k1):
    """A z-slab (vertex planes [k0, k1] of the n x n x nzg mesh) numbers its
    entities as the whole mesh does, shifted: its complete rows of C, M1 and
    M2 are bitwise the whole mesh's (the per-rank assembly of the lattice
    slabs relies on this)."""
    n = 4
    whole = S.TetMesh(n, 0.12, 9, nzg=nzg)
    slab = S.TetMesh(n, 0.12, 9, nzg=nzg, planes=(k0, k1))
    xw, evw, fvw, _ = whole.geometry()
    xs, evs, fvs, _ = slab.geometry()
    nv_plane = (n + 1) ** 2
    assert np.array_equal(xs, xw[k0 * nv_plane:(k1 + 1) * nv_plane])
    # entity id offsets: the whole mesh's ids of the slab's first plane
    eoff = int(np.searchsorted(evw[:, 0], k0 * nv_plane))
    foff = int(np.searchsorted(fvw[:, 0], k0 * nv_plane))
    vsh = k0 * nv_plane
    # (rows whose columns all lie below the slab's top plane: the top plane
    # lacks the edges leaving the slab, so its ids shift, not its order)
    for ops, ents, off, lo, hi in ((("curl", "curl"), (fvs, fvw), (foff, eoff), k0, k1 - 2),
                                   (("mass1", "mass1"), (evs, evw), (eoff, eoff), k0 + 1, k1 - 2),
                                   (("mass2", "mass2"), (fvs, fvw), (foff, foff), k0 + 1, k1 - 2)):
        a, b = getattr(slab, ops[0])(), getattr(whole, ops[1])()
        lo, hi = (0 if k0 == 0 else lo), (k1 if k1 == nzg else hi)
        rows = [r for r in range(a.rows) if lo <= (ents[0][r, 0] + vsh) // nv_plane <= hi]
        assert rows
        for r in rows:
            assert np.array_equal(ents[0][r] + vsh, ents[1][r + off[0]])
            assert np.array_equal(a.row_cols(r) + off[1], b.row_cols(r + off[0])), (ops, r)
            assert np.array_equal(a.row_vals(r), b.row_vals(r + off[0])), (ops, r)
