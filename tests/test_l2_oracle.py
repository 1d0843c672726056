"""CPU: the L^2-error restatement (oracle/l2_oracle.py) used to check the
device Fig. 3 pipeline: the cell rule's exactness, the host projection of
the cavity potential, and first-order convergence of the projection error."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from oracle import l2_oracle as L2
from oracle import tetmesh_oracle as TO


def test_tet_rule_exact_to_degree_5():
    lam, w = L2.tet_rule()
    # int over the unit tet of l1^a l2^b l3^c = a! b! c! / (a + b + c + 3)!
    from math import factorial
    for a, b, c in [(0, 0, 0), (1, 0, 0), (2, 1, 0), (1, 1, 1), (3, 1, 1), (2, 2, 1), (5, 0, 0)]:
        want = factorial(a) * factorial(b) * factorial(c) / factorial(a + b + c + 3)
        got = np.sum(w * lam[:, 1] ** a * lam[:, 2] ** b * lam[:, 3] ** c)
        assert got == pytest.approx(want, rel=1e-13)


@pytest.mark.parametrize("n,mode", [(3, 1), (5, 2)])
def test_host_cavity_projection_matches_numpy(n, mode):
    m, o = S.TetMesh(n, 0.1, 7), TO.OracleTetMesh(n, 0.1, 7)
    assert np.array_equal(m.project_cavity(mode), L2.project_cavity(o, mode))


def test_projection_error_converges_first_order():
    errs = []
    for n in (2, 4, 8):
        o = TO.OracleTetMesh(n, 0.1, 3)
        errs.append(L2.l2_error(o, L2.project_cavity(o, 1), 0, 1)[1])
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(rates > 0.8), (errs, rates)
