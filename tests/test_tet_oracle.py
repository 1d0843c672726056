"""CPU: the C restatement of the 3-D construction (oracle/tet_oracle.c)
against the numpy restatement (oracle/tetmesh_oracle.py, bitwise), against a
numpy least-squares SPAI (tolerance), against the counts of SURVEY.md
Appendix A, and against the product's host builders (bitwise C / M2, Q_sym to
rounding). The C oracle is what the full-size GPU parity tests and the
reference arm of bench.py build their operators with."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200 import configs
from oracle import oracle as O
from oracle import tetmesh_oracle as TO


def _same(a, b):
    return (a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2])
            and np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4]))


def _rows_csr(rows, ncols):
    rp = np.cumsum([0] + [len(r) for r in rows])
    ci = np.array([c for r in rows for c, _ in r], np.int32)
    va = np.array([v for r in rows for _, v in r])
    return (len(rows), ncols, rp, ci, va)


@pytest.mark.parametrize("n,jit,seed", [(2, 0.0, 0), (3, 0.1, 7), (4, 0.15, 11)])
def test_c_oracle_bitwise_equals_numpy_oracle(n, jit, seed):
    r = O.tet_c_operators(n, jit, seed, want=O.TET_OPERATORS)
    o = TO.OracleTetMesh(n, jit, seed)
    ne, nf = len(o.edge_vertices), len(o.face_vertices)
    assert r["counts"][:3] == (ne, nf, len(o.tet_vertices))
    assert _same(r["c"], _rows_csr(o.curl_rows(), ne))
    assert _same(r["d"], _rows_csr(o.div_rows(), nf))
    assert _same(r["m1"], o.mass(1)[0])
    assert _same(r["m2"], o.mass(2)[0])


@pytest.mark.parametrize("n,jit", [(2, 0.1), (3, 0.15)])
def test_c_oracle_spai_matches_lstsq(n, jit):
    r = O.tet_c_operators(n, jit, 5, want=("m1", "q_sym"))
    assert r["counts"][3] == 0
    m1 = r["m1"]
    pat = TO.pattern(m1, "m1")
    cols = TO.spai_lstsq(m1, pat)
    N = m1[0]
    q = np.zeros((N, N))
    for l in range(N):
        q[pat[l], l] = cols[l]
    want = 0.5 * q + 0.5 * q.T
    rows, _, rp, ci, va = r["q_sym"]
    got = np.zeros((N, N))
    got[np.repeat(np.arange(N), np.diff(rp)), ci] = va
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    # Q_sym keeps the (symmetric) S(M1) pattern and is exactly symmetric
    assert np.array_equal(rp, m1[2]) and np.array_equal(ci, m1[3])
    assert np.array_equal(got, got.T)


@pytest.mark.parametrize("n", [5, 16])
def test_c_oracle_counts_match_appendix_a(n):
    r = O.tet_c_operators(n, 0.1, 3, want=("c", "m2", "q_sym"))
    n1, n2, nt, failed = r["counts"]
    assert (n1, n2, nt, failed) == (7 * n**3 - 9 * n**2 + 3 * n, 12 * n**3 + 6 * n**2,
                                    6 * n**3, 0)
    assert r["c"][3].size == 36 * n**3 - 48 * n**2 + 18 * n
    assert r["q_sym"][3].size == 115 * n**3 - 261 * n**2 + 195 * n - 48
    # 84 n^3 + 6 n^2 is the structural count; exact zeros (faces whose
    # element couplings cancel on the unjittered walls) are dropped
    assert 0.99 * (84 * n**3 + 6 * n**2) <= r["m2"][3].size <= 84 * n**3 + 6 * n**2


@pytest.mark.parametrize("n,jit,seed", [(6, 0.15, 2023), (8, 0.1, 5)])
def test_c_oracle_vs_product_host_builders(n, jit, seed):
    r = O.tet_c_operators(n, jit, seed)
    sy = configs.tet_system(n, jit, seed)
    for name, a in (("c", sy.c), ("m2", sy.m2)):
        assert _same(r[name], (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)), name
    q = S.symmetric_part(sy.q)
    b = r["q_sym"]
    assert np.array_equal(b[2], q.row_ptr) and np.array_equal(b[3], q.col_idx)
    assert np.abs(b[4] - q.val).max() <= 1e-13 * np.abs(q.val).max()
