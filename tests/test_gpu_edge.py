"""GPU edge cases the reference's tests exercise for this path: zero steps,
dt = 0, the smallest meshes (one cube; a PEC Yee lattice with no interior
edges), operators with empty rows, a one-DOF system, error contract."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200 import _lib as L
from paper_2301_01753_b200 import configs
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def tup(a):
    return (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)


def test_zero_steps_and_zero_dt_keep_the_state():
    sys_ = configs.tet_system(3, 0.1, seed=1)
    b0, e0, _ = configs.initial_gaussian(sys_, seed=2)
    st = S.make_state(S.Formulation.BE, b0, e0, 1.25)
    s = S.SplitScheme(S.SplitKind.Strang, 0.01, sys_.q, sys_.c, sys_.m2, warn_cfl=False)
    out = s.advance(st, 0)
    assert np.array_equal(out.first, b0) and np.array_equal(out.e, e0) and out.time == 1.25
    z = S.SplitScheme(S.SplitKind.Strang, 0.0, sys_.q, sys_.c, sys_.m2, warn_cfl=False)
    out = z.advance(st, 7)
    assert np.array_equal(out.first, b0) and np.array_equal(out.e, e0)


def test_one_cube_tet_mesh_and_device_scheme():
    """n = 1: one cube, 6 tets; PEC leaves a single interior edge (the body
    diagonal) -- host and device builds agree and the step matches the oracle."""
    mesh = S.TetMesh(1, 0.0, 0)
    assert (mesh.n_edges, mesh.n_faces, mesh.n_tets) == (1, 18, 6)
    sys_ = configs.tet_system(1, 0.0, seed=0)
    dev = S.tet_device_scheme(1, 0.0, seed=0, dt=0.1)
    st = S.make_state(S.Formulation.BE, np.zeros(sys_.n2), np.ones(sys_.n1))
    host = S.SplitScheme(S.SplitKind.Strang, 0.1, sys_.q, sys_.c, sys_.m2, warn_cfl=False)
    a, b = host.advance(st, 5), dev.advance(st, 5)
    np.testing.assert_allclose(b.first, a.first, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(b.e, a.e, rtol=1e-13, atol=1e-15)


def test_pec_lattice_without_interior_edges():
    """1x1x1 PEC: every edge is on the wall, so N1 = 0 and b stays constant."""
    y = S.YeeScheme(1, 1, 1, 1.0, 1.0, 1.0, 0.1, bc=L.BC_PEC)
    assert y.n_edges == 0 and y.n_faces == 6
    b0 = np.arange(1.0, 7.0)
    y.load(b0, np.zeros(0))
    y.advance(10)
    b, e, _ = y.fetch()
    assert np.array_equal(b, b0) and e.size == 0


def test_operator_with_empty_rows_and_one_dof():
    """C with empty rows (boundary faces under PEC) and a 1 x 1 system."""
    q = S.SparseOperator(1, 1, np.array([0, 1]), np.array([0], np.int32), np.array([2.0]), True)
    c = S.SparseOperator(3, 1, np.array([0, 1, 1, 2]), np.array([0, 0], np.int32),
                         np.array([1.0, -1.0]))
    m2 = S.SparseOperator(3, 3, np.array([0, 1, 2, 3]), np.array([0, 1, 2], np.int32),
                          np.array([1.0, 1.0, 1.0]), True)
    b0, e0 = np.array([0.5, 7.0, -0.5]), np.array([0.25])
    s = S.SplitScheme(S.SplitKind.Strang, 0.05, q, c, m2, warn_cfl=False, strict=True)
    out = s.advance(S.make_state(S.Formulation.BE, b0, e0), 9)
    port = O.PortScheme(1, 0.05, tup(q), tup(c), tup(m2), be=True)
    pb, pe, _ = port.steps(b0, e0, 9)
    assert np.array_equal(out.first, pb) and np.array_equal(out.e, pe)
    assert out.first[1] == 7.0  # the empty row keeps its value


def test_error_contract():
    sys_ = configs.tet_system(2, 0.1, seed=1)
    with pytest.raises(L.InvalidParameter):
        S.SplitScheme(S.SplitKind.Strang, -1.0, sys_.q, sys_.c, sys_.m2)
    s = S.SplitScheme(S.SplitKind.Strang, 0.01, sys_.q, sys_.c, sys_.m2, warn_cfl=False)
    with pytest.raises(L.InvalidParameter):
        s.advance(S.make_state(S.Formulation.BE, np.zeros(sys_.n2 + 1), np.zeros(sys_.n1)), 1)
    with pytest.raises(L.InvalidParameter):
        s.curl_of_curl(np.zeros(sys_.n1 + 2))
