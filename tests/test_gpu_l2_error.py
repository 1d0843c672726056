"""GPU: the Fig. 3 accuracy pipeline (reference
operators.cpp:181-257 l2_error, convergence.cpp:107-116) on the Kuhn-tet
Whitney space: canonical projection of the cavity potential A_m, the
curl-of-curl Q C^T M2 C a on the device, and the device L^2 error against
curl curl A_m -- checked against the numpy restatement (oracle/l2_oracle.py)
and for convergence under refinement."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from oracle import l2_oracle as L2
from oracle import tetmesh_oracle as TO

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,kind,mode", [(3, 0, 1), (4, 1, 1), (5, 1, 2)])
def test_device_l2_error_matches_numpy(n, kind, mode):
    m, o = S.TetMesh(n, 0.1, 5), TO.OracleTetMesh(n, 0.1, 5)
    rng = np.random.default_rng(n)
    for w in (m.project_cavity(mode), rng.standard_normal(m.n_edges)):
        got = m.l2_error(w, kind, mode)
        want = L2.l2_error(o, w, kind, mode)
        assert got[0] == pytest.approx(want[0], rel=1e-12)
        assert got[1] == pytest.approx(want[1], rel=1e-12)


def test_fig3_chain_matches_numpy_at_small_size():
    """w = Q C^T M2 C a with a the projected A_1, against the numpy chain on
    the downloaded operators, then the error of both against curl curl A_1"""
    import scipy.sparse as sp
    n = 6
    s = S.tet_device_scheme(n, 0.1, 5)
    m, o = S.TetMesh(n, 0.1, 5), TO.OracleTetMesh(n, 0.1, 5)
    a = m.project_cavity(1)
    w = s.curl_of_curl(a)
    ops = S.tet_device_operators(n, 0.1, 5)
    csr = {k: sp.csr_matrix((v.val, v.col_idx, v.row_ptr), shape=(v.rows, v.cols))
           for k, v in ops.items()}
    want = csr["q_sym"] @ (csr["c"].T @ (csr["m2"] @ (csr["c"] @ a)))
    assert np.abs(w - want).max() <= 1e-12 * np.abs(want).max()
    assert m.l2_error(w, 1, 1)[1] == pytest.approx(L2.l2_error(o, w, 1, 1)[1], rel=1e-12)


def test_fig3_curl_curl_error_converges():
    """the S(M1) SPAI curl-of-curl error against curl curl A_1 falls under
    refinement (Fig. 3's quantity; the paper's 2-D S(M1) slope is ~h^0.73)"""
    errs = []
    for n in (8, 16, 32):
        s = S.tet_device_scheme(n, 0.1, 5)
        m = S.TetMesh(n, 0.1, 5)
        errs.append(m.l2_error(s.curl_of_curl(m.project_cavity(1)), 1, 1)[1])
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    print("relative L2 errors", errs, "rates", rates)
    assert errs[0] > errs[1] > errs[2]
    assert np.all(rates > 0.3)
