"""GPU parity on the unstructured SFEEC path (BASELINE configs 1/3): the B200
step on the tet operators (Whitney P1-, SPAI S(M1), PEC) against the UNMODIFIED
reference SplitScheme (oracle/_ref) fed with the same operators."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200 import configs
from oracle import oracle as O
from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-12


def tup(a):
    return (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)


@pytest.fixture(scope="module")
def cfg1():
    """config 1: 16^3 x 6 tets, jitter 0.1 h, S(M1) SPAI, E0 = 0, B0 = C A, A ~ N(0,1)."""
    sys_ = configs.tet_system(16, 0.1, seed=2023)
    b0, e0, _ = configs.initial_gaussian(sys_, seed=7)
    return sys_, b0, e0


def _reference(sys_, dt, strang=1):
    if O.ref_available():
        return "ref", O.RefScheme(strang, dt, tup(sys_.q), tup(sys_.c), tup(sys_.m2),
                                  div=tup(sys_.d))
    return "port", O.PortScheme(strang, dt, tup(sys_.q), tup(sys_.c), tup(sys_.m2),
                                div=tup(sys_.d))


def _ref_steps(kind, ref, b0, e0, n):
    if kind == "ref":
        b, e, _, hist = ref.steps(True, b0, e0, n, energy=True)
    else:
        b, e, hist = ref.steps(b0, e0, n, energy=True)
    return b, e, hist


def test_config1_cfl_and_100_steps_match_reference(cfg1):
    sys_, b0, e0 = cfg1
    s = S.SplitScheme(S.SplitKind.Strang, 1.0, sys_.q, sys_.c, sys_.m2, div=sys_.d,
                      warn_cfl=False)
    kind, ref1 = _reference(sys_, 1.0)
    nu_dev, nu_ref = s.cfl_number(), ref1.cfl()
    assert nu_dev == pytest.approx(nu_ref, rel=1e-10)
    dt = configs.cfl_dt(s)
    s.set_dt(dt)
    assert s.cfl_number() == pytest.approx(1.0, rel=1e-12)  # nu = 1 at 0.5 dt_CFL
    kind, ref = _reference(sys_, dt)
    rb, re, rh = _ref_steps(kind, ref, b0, e0, 100)
    out, en, gauss = s.advance_diag(S.make_state(S.Formulation.BE, b0, e0), 100, 1)
    assert rel_l2(out.first, rb) <= TOL
    assert rel_l2(out.e, re) <= TOL
    assert np.max(np.abs(en - rh)) <= TOL * rh[0]
    # energy drift of the symplectic scheme stays bounded and matches the oracle's
    drift_dev = (en.max() - en.min()) / en[0]
    drift_ref = (rh.max() - rh.min()) / rh[0]
    assert drift_dev == pytest.approx(drift_ref, rel=1e-6, abs=1e-13)
    # B0 = C A is discretely divergence free and stays so (test_dynamics.cpp:286-299)
    assert np.max(gauss) <= 1e-12 * np.max(np.abs(b0))


def test_config1_strict_mode_bitwise(cfg1):
    sys_, b0, e0 = cfg1
    dt = 0.01
    s = S.SplitScheme(S.SplitKind.Strang, dt, sys_.q, sys_.c, sys_.m2, warn_cfl=False,
                      strict=True)
    kind, ref = _reference(sys_, dt)
    rb, re, _ = _ref_steps(kind, ref, b0, e0, 20)
    out = s.advance(S.make_state(S.Formulation.BE, b0, e0), 20)
    assert np.array_equal(out.first, rb) and np.array_equal(out.e, re)


@pytest.mark.parametrize("strang", [1, 0])
def test_pulse_init_both_splittings(strang):
    """config-3 style Gaussian pulse on a small mesh (jitter 0.15 h)."""
    sys_ = configs.tet_system(10, 0.15, seed=5)
    b0, e0, _ = configs.initial_pulse(sys_, seed=3)
    dt = 0.002
    s = S.SplitScheme(strang, dt, sys_.q, sys_.c, sys_.m2, warn_cfl=False)
    kind, ref = _reference(sys_, dt, strang)
    rb, re, rh = _ref_steps(kind, ref, b0, e0, 60)
    out = s.advance(S.make_state(S.Formulation.BE, b0, e0), 60)
    assert rel_l2(out.first, rb) <= TOL and rel_l2(out.e, re) <= TOL


def test_layouts_selected_and_timing_reported(cfg1):
    sys_, b0, e0 = cfg1
    s = S.SplitScheme(S.SplitKind.Strang, 0.01, sys_.q, sys_.c, sys_.m2, warn_cfl=False)
    s.load(S.make_state(S.Formulation.BE, b0, e0))
    s.kernel_timing(True)
    out = s.advance(S.make_state(S.Formulation.BE, b0, e0), 10)
    t = s.kernel_timing(False)
    assert t["K-Q"]["launches"] == 11 and t["K-M2"]["launches"] == 10
    assert all(t[k]["ms"] > 0 for k in ("K-Q", "K-Cb", "K-CTe", "K-M2"))
    assert s.last_launches() == 4 * 10 + 2
    assert np.isfinite(out.first).all()
