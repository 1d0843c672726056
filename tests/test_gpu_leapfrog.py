"""GPU parity of the unstructured leapfrog (C ABI -> sm_100a kernels) against
the oracle and the reference's golden fixtures, plus the reference's own
dynamics properties (test_dynamics.cpp) restated on the device."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200 import _lib as L
from oracle import oracle as O
from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-12  # BASELINE.json north_star: fp64 E/B within 1e-12 relative L2


def _ops(g):
    n1, n2 = int(g["n1"]), int(g["n2"])
    q = S.SparseOperator(n1, n1, g["q_rp"], g["q_ci"], g["q_va"])
    c = S.SparseOperator(n2, n1, g["c_rp"], g["c_ci"], g["c_va"])
    m2 = S.SparseOperator(n2, n2, g["m2_rp"], g["m2_ci"], g["m2_va"], True)
    return q, c, m2


@pytest.mark.parametrize("strang", [1, 0])
@pytest.mark.parametrize("be", [1, 0])
def test_strict_mode_is_bitwise_reference(golden, strang, be):
    g = golden("scheme.npz")
    q, c, m2 = _ops(g)
    key = f"s{strang}b{be}"
    form = S.Formulation.BE if be else S.Formulation.AE
    s = S.SplitScheme(strang, 0.05, q, c, m2, warn_cfl=False, formulation=form, strict=True)
    first0 = g["b0"] if be else g["a0"]
    out = s.advance(S.make_state(form, first0, g["e0"]), 20)
    assert np.array_equal(out.first, g[f"{key}_first"])
    assert np.array_equal(out.e, g[f"{key}_e"])
    assert out.time == g[f"{key}_t"]
    st = S.make_state(form, first0, g["e0"])
    s.flow_he(st, 0.34)
    assert np.array_equal(st.first, g[f"{key}_flowhe_first"])
    assert np.array_equal(st.e, g[f"{key}_flowhe_e"])
    st = S.make_state(form, first0, g["e0"])
    s.flow_ha(st, 0.7)
    assert np.array_equal(st.first, g[f"{key}_flowha_first"])
    assert np.array_equal(st.e, g[f"{key}_flowha_e"])
    qs = s.q_sym()
    assert np.array_equal(qs.val, g["qsym_va"]) and np.array_equal(qs.col_idx, g["qsym_ci"])


@pytest.mark.parametrize("strang", [1, 0])
@pytest.mark.parametrize("be", [1, 0])
def test_production_mode_within_tolerance(golden, strang, be):
    g = golden("scheme.npz")
    q, c, m2 = _ops(g)
    key = f"s{strang}b{be}"
    form = S.Formulation.BE if be else S.Formulation.AE
    s = S.SplitScheme(strang, 0.05, q, c, m2, warn_cfl=False, formulation=form)
    first0 = g["b0"] if be else g["a0"]
    out, energy, _ = s.advance_diag(S.make_state(form, first0, g["e0"]), 20, 1)
    assert rel_l2(out.first, g[f"{key}_first"]) <= TOL
    assert rel_l2(out.e, g[f"{key}_e"]) <= TOL
    assert np.max(np.abs(energy - g[f"{key}_energy"])) <= TOL * abs(g[f"{key}_energy0"])
    assert s.cfl_number() == pytest.approx(float(g[f"{key}_cfl"]), rel=1e-10)


def _cubical_system(n=2):
    """Yee-PEC lattice C with synthetic SPD M2 and a nonsymmetric Q."""
    from tests.golden.make_golden import synthetic_ops
    q, c, m2, cs = synthetic_ops(n=n, seed=1)
    to = lambda a, sym=False: S.SparseOperator(a[0], a[1], a[2], a[3], a[4], sym)
    return to(q), to(c), to(m2, True), cs


def test_subflow_closed_forms():
    """test_dynamics.cpp:67-94 on the device (exact)."""
    q, c, m2, _ = _cubical_system()
    n1 = c.cols
    s = S.SplitScheme(S.SplitKind.Strang, 0.1, q, c, m2, formulation=S.Formulation.AE)
    rnd = lambda seed: O.port_uniform(seed, n1)
    st = S.make_state(S.Formulation.AE, rnd(1), np.zeros(n1))
    a = st.first.copy()
    s.flow_he(st, 0.34)
    assert np.array_equal(st.first, a)
    st = S.make_state(S.Formulation.AE, rnd(2), rnd(3))
    a, e = st.first.copy(), st.e.copy()
    s.flow_he(st, 0.0)
    s.flow_ha(st, 0.0)
    assert np.array_equal(st.first, a) and np.array_equal(st.e, e)
    st = S.make_state(S.Formulation.AE, np.zeros(n1), rnd(4))
    e = st.e.copy()
    s.flow_ha(st, 0.7)
    assert np.array_equal(st.e, e)


def test_scalar_toy_flow():
    """test_dynamics.cpp:96-111."""
    q = S.scaled_identity(1, 1.0 / 2.0)
    c = S.SparseOperator(1, 1, [0, 0], [], [])
    m2 = S.scaled_identity(1, 1.0)
    s = S.SplitScheme(S.SplitKind.Strang, 0.25, q, c, m2, warn_cfl=False,
                      formulation=S.Formulation.AE)
    st = S.make_state(S.Formulation.AE, [1.0], [0.5])
    s.flow_he(st, 0.25)
    assert st.first[0] == pytest.approx(1.0 - 0.25 * 0.5 / 2.0, rel=1e-15)
    assert st.e[0] == 0.5 and st.time == 0.0


def test_zero_state_stays_zero_and_clock():
    """test_dynamics.cpp:137-148."""
    q, c, m2, _ = _cubical_system()
    s = S.SplitScheme(S.SplitKind.Strang, 0.1, q, c, m2, formulation=S.Formulation.AE)
    z = S.make_state(S.Formulation.AE, np.zeros(c.cols), np.zeros(c.cols))
    out = z
    for _ in range(50):
        out = s.step(out)
    assert s.energy(out) == 0.0
    assert not out.first.any() and not out.e.any()
    assert out.time == pytest.approx(5.0)


def test_strang_local_error_is_third_order():
    """test_dynamics.cpp:150-170: one step vs two half steps ratio ~ 8."""
    q, c, m2, _ = _cubical_system()
    n1 = c.cols
    f0, e0 = O.port_uniform(7, n1), O.port_uniform(8, n1)

    def dev(dt):
        full = S.SplitScheme(S.SplitKind.Strang, dt, q, c, m2, warn_cfl=False,
                             formulation=S.Formulation.AE)
        half = S.SplitScheme(S.SplitKind.Strang, dt / 2, q, c, m2, warn_cfl=False,
                             formulation=S.Formulation.AE)
        a = full.step(S.make_state(S.Formulation.AE, f0, e0))
        b = half.advance(S.make_state(S.Formulation.AE, f0, e0), 2)
        return max(np.max(np.abs(a.first - b.first)), np.max(np.abs(a.e - b.e)))

    d1, d2, d3 = dev(0.1), dev(0.05), dev(0.025)
    assert d1 / d2 == pytest.approx(8.0, rel=0.3)
    assert d2 / d3 == pytest.approx(8.0, rel=0.3)


def test_gauss_residual_preserved_pec_yee():
    """test_dynamics.cpp:286-311 on a PEC lattice with D from the builder."""
    c, d = S.yee_operators(3, 3, 3, 1.0, 0.5, 2.0, bc=L.BC_PEC)
    dv = 1.0 * 0.5 * 2.0
    q = S.scaled_identity(c.cols, 1.0 / dv)
    m2 = S.scaled_identity(c.rows, dv)
    s = S.SplitScheme(S.SplitKind.Strang, 0.05, q, c, m2, div=d, warn_cfl=False)
    a0 = O.port_uniform(20, c.cols)
    b0 = c.to_dense() @ a0
    st = S.make_state(S.Formulation.BE, b0, O.port_uniform(21, c.cols))
    assert s.gauss_residual(st) <= 1e-14
    out = s.advance(st, 2000)
    assert s.gauss_residual(out) <= 1e-13
    t = S.make_state(S.Formulation.BE, O.port_uniform(22, c.rows), O.port_uniform(23, c.cols))
    r0 = s.gauss_residual(t)
    assert r0 > 0.1
    out = s.advance(t, 500)
    assert s.gauss_residual(out) == pytest.approx(r0, rel=1e-13)
    with pytest.raises(S.InvalidParameter):
        s.gauss_residual(S.make_state(S.Formulation.AE, a0, a0))


def test_cfl_linear_in_dt():
    """test_dynamics.cpp:332-340."""
    q, c, m2, _ = _cubical_system()
    s1 = S.SplitScheme(S.SplitKind.Strang, 0.1, q, c, m2, warn_cfl=False)
    s2 = S.SplitScheme(S.SplitKind.Strang, 0.2, q, c, m2, warn_cfl=False)
    assert s1.cfl_number() > 0
    assert s2.cfl_number() == pytest.approx(2 * s1.cfl_number(), rel=1e-10)


def test_device_matches_live_oracle_larger_pec():
    """PEC lattice 6x5x7 with lumped masses: production device vs the port
    after 100 steps and the energy history (sizes the oracle does in <1 s)."""
    c, d = S.yee_operators(6, 5, 7, 1.0, 0.8, 1.25, bc=L.BC_PEC)
    dv = 1.0 * 0.8 * 1.25
    q = S.scaled_identity(c.cols, 1.0 / dv)
    m2 = S.scaled_identity(c.rows, dv)
    tup = lambda a: (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)
    a0 = O.port_uniform(3, c.cols)
    b0 = O.port_spmv(tup(c), a0)
    e0 = np.zeros(c.cols)
    port = O.PortScheme(1, 0.2, tup(q), tup(c), tup(m2), be=True)
    pf, pe, ph = port.steps(b0, e0, 100, energy=True)
    s = S.SplitScheme(S.SplitKind.Strang, 0.2, q, c, m2, warn_cfl=False)
    out, en, _ = s.advance_diag(S.make_state(S.Formulation.BE, b0, e0), 100, 1)
    assert rel_l2(out.first, pf) <= TOL and rel_l2(out.e, pe) <= TOL
    assert np.max(np.abs(en - ph)) <= TOL * ph[0]


@pytest.mark.parametrize("strang", [1, 0])
def test_non_default_units_match_reference(strang):
    """UnitSystem{eps0, mu0} != 1 (dynamics.hpp:9-18): c^2 = 1/(eps0 mu0) in the
    e-kick and eps0 / mu0 weights in the energy -- strict mode bitwise the
    reference step, production within 1e-12, energy and CFL to round-off."""
    from paper_2301_01753_b200 import configs
    sys_ = configs.tet_system(4, 0.1, seed=6)
    b0, e0, _ = configs.initial_gaussian(sys_, seed=3)
    tup = lambda a: (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)  # noqa: E731
    units = S.UnitSystem(eps0=2.5, mu0=0.4)
    dt, steps = 0.02, 30
    kind = S.SplitKind.Strang if strang else S.SplitKind.LieTrotter
    if O.ref_available():
        ref = O.RefScheme(strang, dt, tup(sys_.q), tup(sys_.c), tup(sys_.m2), eps0=2.5, mu0=0.4)
        rb, re_, _, _ = ref.steps(True, b0, e0, steps)
        r_energy = ref.energy(True, rb, re_)
        r_cfl = ref.cfl()
    else:
        port = O.PortScheme(strang, dt, tup(sys_.q), tup(sys_.c), tup(sys_.m2), eps0=2.5, mu0=0.4)
        rb, re_, _ = port.steps(b0, e0, steps)
        r_energy = port.energy(rb, re_)
        r_cfl = port.cfl()
    for strict in (True, False):
        s = S.SplitScheme(kind, dt, sys_.q, sys_.c, sys_.m2, units=units, warn_cfl=False,
                          strict=strict)
        out = s.advance(S.make_state(S.Formulation.BE, b0, e0), steps)
        if strict:
            assert np.array_equal(out.first, rb) and np.array_equal(out.e, re_)
        else:
            assert rel_l2(out.first, rb) <= TOL and rel_l2(out.e, re_) <= TOL
        assert s.energy(out) == pytest.approx(r_energy, rel=1e-13)
        assert s.cfl_number() == pytest.approx(r_cfl, rel=1e-10)
