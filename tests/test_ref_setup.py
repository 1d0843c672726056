"""The product's setup producers against the reference's OWN setup code.

oracle/_ref/libsfeec_ref_setup.so is the whole unmodified reference library
(form_space.cpp, operators.cpp, spai.cpp included) compiled over the
Eigen-subset stand-in oracle/eigen_shim. It answers VERDICT
r1's "parity unpinned by the reference" for what the reference does define:

  * make_pattern (spai.cpp:31-72): the product's S(M1) / S(M1^2) patterns of
    the 3-D tet M1 (first and second order) are index-for-index the
    reference's;
  * spai_approximate_inverse (spai.cpp:127-286): the product's SPAI values
    match the reference's on the same M1 (the dense solves differ in
    elimination order, hence the tolerance);
  * mass_matrix / derivative_matrix (operators.cpp:111-179) of the Q1 cubical
    lattice: the product's periodic Yee masses and curl are bitwise the
    reference's.
The library is built where /root/reference exists and travels prebuilt."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.refsetup_available(),
                                reason="oracle/_ref/libsfeec_ref_setup.so not built")


def tup(a):
    return (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)


def same_pattern(a, b):
    return (a[0] == b.rows and np.array_equal(a[2], b.row_ptr)
            and np.array_equal(a[3], b.col_idx))


def tet_m1(order, n, jitter=0.1, seed=4):
    m = S.TetMesh(n, jitter, seed)
    return m.mass1() if order == 1 else m.p2_operator("m1")


@pytest.mark.parametrize("order,n,kind", [(1, 4, "diagonal"), (1, 4, "m1"), (1, 4, "m1sq"),
                                          (1, 6, "m1"), (2, 2, "m1"), (2, 2, "m1sq"),
                                          (2, 3, "m1sq")])
def test_pattern_is_the_references(order, n, kind):
    m1 = tet_m1(order, n)
    assert same_pattern(O.ref_make_pattern(tup(m1), kind), S.make_pattern(m1, kind))


@pytest.mark.parametrize("order,n,kind", [(1, 4, "diagonal"), (1, 4, "m1"), (1, 5, "m1sq"),
                                          (1, 6, "m1"), (2, 2, "m1"), (2, 2, "m1sq")])
def test_spai_values_match_the_references(order, n, kind):
    m1 = tet_m1(order, n)
    q, rep = S.spai_approximate_inverse(m1, kind)
    rq, rrep = O.ref_spai(tup(m1), kind)
    assert same_pattern(rq, q)  # operator_from_triplets keeps the pattern (no exact zeros)
    scale = np.abs(rq[4]).max()
    assert np.max(np.abs(q.val - rq[4])) <= 1e-11 * scale
    assert rep["fallback_columns"] == rrep["fallback_columns"] == 0
    assert rep["frobenius_residual"] == pytest.approx(rrep["frobenius_residual"], rel=1e-9)
    assert rep["max_column_residual"] == pytest.approx(rrep["max_column_residual"], rel=1e-9)
    # and the reference's CG path (test_spai.cpp:203-214) lands on the same Q
    cq, _ = O.ref_spai(tup(m1), kind, use_cg=True)
    assert np.max(np.abs(q.val - cq[4])) <= 1e-8 * scale


def test_q_sym_of_the_step_is_the_references():
    """Q_sym as the step uses it: symmetric_part of the reference's SPAI of the
    tet M1 against the product's, entry by entry."""
    m1 = tet_m1(1, 5)
    q, _ = S.spai_approximate_inverse(m1, "m1")
    rq, _ = O.ref_spai(tup(m1), "m1")
    got = S.symmetric_part(q)
    want = O.port_symmetric_part(rq) if hasattr(O, "port_symmetric_part") else None
    assert want is not None
    assert np.array_equal(got.row_ptr, want[2]) and np.array_equal(got.col_idx, want[3])
    assert np.max(np.abs(got.val - want[4])) <= 1e-11 * np.abs(want[4]).max()


@pytest.mark.parametrize("dims,d", [((3, 4, 5), (0.5, 1.0, 2.0)), ((2, 2, 3), (0.3, 0.7, 1.1)),
                                    ((4, 4, 4), (1.0, 1.0, 1.0))])
def test_cubical_operators_bitwise_the_references(dims, d):
    """Periodic Q1 lattice: the product's masses (host_yee.cpp build_yee_mass)
    and curl / divergence are bit for bit the reference's mass_matrix and
    derivative_matrix on the reference's own mesh and spaces."""
    m1, m2 = S.yee_masses(*dims, *d, bc=0)
    c, dv = S.yee_operators(*dims, *d, bc=0)
    for name, got in (("m1", m1), ("m2", m2), ("c", c), ("d", dv)):
        want = O.ref_cubical_operator(*dims, *d, name)
        assert same_pattern(want, got), name
        assert np.array_equal(want[4], got.val), name


def test_cubical_spai_matches_the_references():
    """test_dynamics.cpp's cubical_system: S(M1) SPAI of the consistent Q1 M1."""
    m1, _ = S.yee_masses(3, 3, 3, 1.0, 0.7, 1.3, bc=0)
    q, _ = S.spai_approximate_inverse(m1, "m1")
    rq, _ = O.ref_spai(tup(m1), "m1")
    assert same_pattern(rq, q)
    assert np.max(np.abs(q.val - rq[4])) <= 1e-12 * np.abs(rq[4]).max()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [5, 8])
def test_device_assembled_q_sym_is_the_references(n):
    """The device-assembled Q_sym of the tet system (tet_device.cu: one warp
    per SPAI column, Cholesky in shared memory) against symmetric_part of the
    reference's own SPAI of the same M1."""
    ops = S.tet_device_operators(n, 0.1, 2023)
    m1 = S.TetMesh(n, 0.1, 2023).mass1()
    rq, rep = O.ref_spai(tup(m1), "m1")
    assert rep["fallback_columns"] == 0
    want = O.port_symmetric_part(rq)
    got = ops["q_sym"]
    assert np.array_equal(got.row_ptr, want[2]) and np.array_equal(got.col_idx, want[3])
    assert np.max(np.abs(got.val - want[4])) <= 1e-11 * np.abs(want[4]).max()


@pytest.mark.gpu
def test_device_p2_spai_is_the_references():
    """The S(M1^2) SPAI of the second-order M1 on the device (p2_device.cu: one
    CTA per column, blocked Cholesky) against the reference's."""
    m1 = S.TetMesh(2, 0.1, 3).p2_operator("m1")
    q, fb = S.spai_device(m1)
    rq, rep = O.ref_spai(tup(m1), "m1sq")
    assert fb == 0 and rep["fallback_columns"] == 0
    assert same_pattern(rq, q)
    assert np.max(np.abs(q.val - rq[4])) <= 1e-10 * np.abs(rq[4]).max()
