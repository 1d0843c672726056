"""Consistent Q1- masses of the cubical lattice (reference mass_matrix,
operators.cpp:133-179): the reference's golden table (test_operators.cpp:110-149),
bitwise against the oracle restatement, the S(M1) pattern of 9 entries per row
(test_spai.cpp:94), and PEC (new: boundary edges dropped)."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2301_01753_b200 as S
from oracle import cubical_oracle as CO


def _csr(a):
    return sp.csr_matrix((a.val, a.col_idx, a.row_ptr), shape=(a.rows, a.cols))


def test_golden_table():
    dx, dy, dz = 0.5, 1.0, 2.0
    dv = dx * dy * dz
    m1, m2 = (_csr(m) for m in S.yee_masses(3, 3, 3, dx, dy, dz, bc=0))
    N = 27
    vid = lambda i, j, k: i + 3 * (j + 3 * k)  # noqa: E731
    e = vid(1, 1, 1)
    assert m1[e, e] == pytest.approx(4 * dv / 9, rel=1e-13)
    assert m1[e, vid(1, 2, 1)] == pytest.approx(dv / 9, rel=1e-13)
    assert m1[e, vid(1, 1, 2)] == pytest.approx(dv / 9, rel=1e-13)
    assert m1[e, vid(1, 2, 2)] == pytest.approx(dv / 36, rel=1e-13)
    assert m1[e, vid(1, 0, 2)] == pytest.approx(dv / 36, rel=1e-13)
    assert m1[e, N + vid(1, 1, 1)] == 0.0
    assert m2[e, e] == pytest.approx(2 * dv / 3, rel=1e-13)
    assert m2[e, vid(2, 1, 1)] == pytest.approx(dv / 6, rel=1e-13)
    assert m2[e, vid(0, 1, 1)] == pytest.approx(dv / 6, rel=1e-13)
    for m in (m1, m2):
        np.testing.assert_allclose(np.asarray(m.sum(axis=1)).ravel(), dv, rtol=1e-13)
    # wrap-around merging on a 2-lattice keeps row sums
    small, _ = S.yee_masses(2, 2, 2, 1, 1, 1, bc=0)
    np.testing.assert_allclose(np.asarray(_csr(small).sum(axis=1)).ravel(), 1.0, rtol=1e-13)


@pytest.mark.parametrize("dims,d", [((3, 4, 5), (0.5, 1.0, 2.0)), ((2, 2, 3), (0.3, 0.7, 1.1)),
                                    ((1, 3, 2), (1.0, 1.0, 1.0))])
def test_bitwise_equals_oracle(dims, d):
    for form, m in zip((1, 2), S.yee_masses(*dims, *d, bc=0)):
        rows = CO.mass_periodic(*dims, *d, form)
        assert m.rows == len(rows)
        for r, row in enumerate(rows):
            cols = m.col_idx[m.row_ptr[r]:m.row_ptr[r + 1]]
            vals = m.val[m.row_ptr[r]:m.row_ptr[r + 1]]
            assert [c for c, _ in row] == list(cols)
            assert np.array_equal(np.array([v for _, v in row]), vals)


def test_spai_pattern_and_pec():
    m1, _ = S.yee_masses(4, 4, 4, 1.0, 1.0, 1.0, bc=0)
    assert set(np.diff(S.make_pattern(m1, "m1").row_ptr)) == {9}
    m1p, m2p = S.yee_masses(4, 3, 5, 0.7, 1.0, 1.3, bc=1)
    c, _ = S.yee_operators(4, 3, 5, 0.7, 1.0, 1.3, bc=1)
    assert (m1p.rows, m2p.rows) == (c.cols, c.rows)
    for m in (m1p, m2p):
        a = _csr(m)
        assert (a != a.T).nnz == 0
        assert np.linalg.eigvalsh(a.toarray()).min() > 0
