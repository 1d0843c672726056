"""GPU: the second-order P2^- system with the S(M1^2) SPAI (BASELINE config
4). The device SPAI (blocked Cholesky per column, p2_device.cu) against the
host SPAI (unblocked Cholesky, spai.cpp:127-286 restated) and a numpy least-
squares solve; the device-built operators against the host builders; the
leapfrog on them against the C oracle step; Gauss law and energy."""
import time

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2301_01753_b200 as S
from oracle import oracle as O
from paper_2301_01753_b200 import configs, inputs
from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu


def tup(a):
    return (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)


def csr(a):
    return sp.csr_matrix((a.val, a.col_idx, a.row_ptr), shape=(a.rows, a.cols))


def same(a, b):
    return (a.rows == b.rows and a.cols == b.cols and np.array_equal(a.row_ptr, b.row_ptr)
            and np.array_equal(a.col_idx, b.col_idx) and np.array_equal(a.val, b.val))


@pytest.mark.parametrize("n,seed", [(2, 4), (4, 11)])
def test_device_spai_matches_host_spai(n, seed):
    m1 = S.TetMesh(n, 0.1, seed).p2_operator("m1")
    qd, fb = S.spai_device(m1)
    qh, rep = S.spai_approximate_inverse(m1, "m1sq")
    assert fb == 0 and rep["fallback_columns"] == 0
    assert np.array_equal(qd.row_ptr, qh.row_ptr) and np.array_equal(qd.col_idx, qh.col_idx)
    assert np.abs(qd.val - qh.val).max() <= 1e-10 * np.abs(qh.val).max()
    # and a least-squares solve of a few columns
    M = csr(m1).toarray()
    Q = csr(qd).toarray()
    P = csr(S.make_pattern(m1, "m1sq"))
    for l in range(0, M.shape[0], max(1, M.shape[0] // 15)):
        I = P[l].indices
        x, *_ = np.linalg.lstsq(M[:, I], np.eye(M.shape[0])[:, l], rcond=None)
        assert np.abs(Q[I, l] - x).max() <= 1e-9 * max(1.0, np.abs(x).max())


def test_device_operators_match_host_builders():
    n, jit, seed = 3, 0.1, 5
    mesh = S.TetMesh(n, jit, seed)
    dev = S.p2_device_operators(n, jit, seed)
    c = mesh.p2_operator("c")
    assert same(dev["c"], c)
    assert same(dev["m2"], mesh.p2_operator("m2"))
    assert same(dev["d"], mesh.p2_operator("d"))
    assert same(dev["ct"], S.transpose(c))
    q, _ = S.spai_approximate_inverse(mesh.p2_operator("m1"), "m1sq")
    qs = S.symmetric_part(q)
    a = dev["q_sym"]
    assert np.array_equal(a.row_ptr, qs.row_ptr) and np.array_equal(a.col_idx, qs.col_idx)
    assert np.abs(a.val - qs.val).max() <= 1e-10 * np.abs(qs.val).max()
    assert (csr(a) != csr(a).T).nnz == 0  # exactly symmetric


@pytest.fixture(scope="module")
def p2_small():
    n, jit, seed = 6, 0.1, 2023
    s = S.p2_device_scheme(n, jit, seed, dt=1.0, with_div=True)
    a = inputs.gaussian(7, s._n1)
    b0 = s.apply("c", a)
    s.set_dt(configs.cfl_dt(s))
    return n, jit, seed, s, b0, np.zeros(s._n1)


def test_p2_scheme_steps_like_the_oracle(p2_small):
    n, jit, seed, s, b0, e0 = p2_small
    ops = S.p2_device_operators(n, jit, seed)
    port = O.PortScheme(1, s.dt(), tup(ops["q_sym"]), tup(ops["c"]), tup(ops["m2"]),
                        q_is_symmetric=True)
    pb, pe, _ = port.steps(b0, e0, 40)
    out = s.advance(S.make_state(S.Formulation.BE, b0, e0), 40)
    assert rel_l2(out.first, pb) <= 1e-12 and rel_l2(out.e, pe) <= 1e-12


def test_p2_gauss_energy_and_cfl(p2_small):
    n, jit, seed, s, b0, e0 = p2_small
    out, en, gauss = s.advance_diag(S.make_state(S.Formulation.BE, b0, e0), 400, 20)
    assert np.max(gauss) <= 1e-12 * np.abs(b0).max()
    assert (en.max() - en.min()) / en[0] <= 0.05
    assert s.cfl_number() == pytest.approx(1.0, rel=1e-9)


def test_p2_pattern_counts_and_setup_time():
    """nnz of the S(M1^2) pattern at n = 12 against the App. A fit (exact
    zeros dropped from M1 can only remove entries), and the setup time."""
    n = 12
    t0 = time.perf_counter()
    s = S.p2_device_scheme(n, 0.1, 2023, dt=1.0)
    dt = time.perf_counter() - t0
    fit = 12028 * n**3 - 30588 * n**2 + 26748 * n - 8208
    assert s._n1 == 38 * n**3 - 30 * n**2 + 6 * n and s._n2 == 54 * n**3 + 18 * n**2
    assert 0.999 * fit <= s.nnz_q <= fit
    print(f"\np2 n={n}: N1={s._n1} nnz(Q)={s.nnz_q} setup {dt:.2f} s")
