"""GPU parity of the structured lumped-mass (Yee) path: periodic against the
reference FDTD and lumped SplitScheme fixtures, PEC against the oracle step on
the builder's CSR operators, fused vs unfused kernels, fp32 vs fp64."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200 import _lib as L
from oracle import oracle as O
from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-12


def test_periodic_matches_reference_fixture(golden):
    """yee_equivalence_check recipe (yee.cpp:83-135): device vs the reference's
    lumped SplitScheme and FDTD on 3x4x5 (1, .5, 2), dt .15, 60 steps."""
    g = golden("yee.npz")
    nx, ny, nz = (int(v) for v in g["dims"])
    d, dt, steps = [float(v) for v in g["d"]], float(g["dt"]), int(g["steps"])
    dv = d[0] * d[1] * d[2]
    y = S.YeeScheme(nx, ny, nz, *d, dt, bc=L.BC_PERIODIC)
    y.load(g["bgrid0"] / dv, g["e0"])
    y.advance(steps)
    b, e, t = y.fetch()
    assert rel_l2(e, g["e_sfeec"]) <= TOL and rel_l2(b, g["b_sfeec"]) <= TOL
    assert t == pytest.approx(float(g["t"]), rel=0, abs=1e-12)
    y.flow_he(0.5 * dt)
    bh, eh, _ = y.fetch()
    assert np.max(np.abs(eh - g["e_fdtd"])) <= 1e-12
    assert np.max(np.abs(dv * bh - g["b_fdtd"])) <= 1e-12


def _pec_case(nx, ny, nz, d, dt, steps, seed=3):
    c, dm = S.yee_operators(nx, ny, nz, *d, bc=L.BC_PEC)
    dv = d[0] * d[1] * d[2]
    tup = lambda a: (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)
    n1, n2 = c.cols, c.rows
    q = (n1, n1, np.arange(n1 + 1), np.arange(n1, dtype=np.int32), np.full(n1, 1.0 / dv))
    m2 = (n2, n2, np.arange(n2 + 1), np.arange(n2, dtype=np.int32), np.full(n2, dv))
    a0 = O.port_uniform(seed, n1)
    b0 = O.port_spmv(tup(c), a0)
    e0 = O.port_uniform(seed + 1, n1)
    port = O.PortScheme(1, dt, q, tup(c), m2, be=True, div=tup(dm))
    pb, pe, ph = port.steps(b0, e0, steps, energy=True)
    return b0, e0, pb, pe, ph, port


@pytest.mark.parametrize("variant", [0, 1, 2, 4])
@pytest.mark.parametrize("dims", [(6, 5, 7), (33, 9, 40), (40, 17, 3), (64, 16, 65)])
def test_pec_matches_oracle(variant, dims):
    d = (1.0, 0.8, 1.25)
    steps = 50
    b0, e0, pb, pe, ph, port = _pec_case(*dims, d, 0.2, steps)
    y = S.YeeScheme(*dims, *d, 0.2, bc=L.BC_PEC)
    y.set_variant(variant)
    y.load(b0, e0)
    y.advance(steps)
    b, e, _ = y.fetch()
    assert rel_l2(b, pb) <= TOL and rel_l2(e, pe) <= TOL
    assert y.energy() == pytest.approx(ph[-1], rel=TOL)
    assert port.gauss(b) <= 1e-12


def test_fused_equals_unfused_closely():
    dims, d = (37, 21, 70), (1.0, 1.0, 1.0)
    rng = np.random.default_rng(0)
    ys = []
    for v in (0, 1, 2, 4):
        y = S.YeeScheme(*dims, *d, 0.3, bc=L.BC_PEC)
        y.set_variant(v)
        if not ys:
            b0, e0 = rng.standard_normal(y.n_faces), rng.standard_normal(y.n_edges)
        y.load(b0, e0)
        y.advance(25)
        ys.append(y.fetch())
    for k in (1, 2, 3):
        assert rel_l2(ys[k][0], ys[0][0]) <= 1e-14 and rel_l2(ys[k][1], ys[0][1]) <= 1e-14


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("steps", [1, 2, 3, 8, 11])
def test_two_step_sweep_equals_single_step_sweeps(prec, steps):
    """Variant 4 (two leapfrog steps per z-sweep, E1/B1/E2 kept on chip) runs
    the same per-point expressions as variant 2: bitwise equal, for odd and
    even step counts and ragged tiles / chunks."""
    dims, d = (45, 19, 70), (1.0, 0.9, 1.1)
    rng = np.random.default_rng(1)
    out = {}
    for v in (2, 4):
        y = S.YeeScheme(*dims, *d, 0.25, bc=L.BC_PEC, precision=prec)
        y.set_variant(v)
        if not out:
            b0, e0 = rng.standard_normal(y.n_faces), rng.standard_normal(y.n_edges)
        y.load(b0, e0)
        y.advance(steps)
        out[v] = y.fetch()
    assert np.array_equal(out[2][0], out[4][0]) and np.array_equal(out[2][1], out[4][1])


def test_fp32_tracks_fp64():
    """fp32 fields (config 2): relative L2 vs fp64 after 200 steps and energy
    drift are reported; bound set from measurement."""
    dims, d = (24, 20, 28), (1.0, 1.0, 1.0)
    out = {}
    for prec in (8, 4):
        y = S.YeeScheme(*dims, *d, 0.25, bc=L.BC_PEC, precision=prec)
        c, _ = S.yee_operators(*dims, *d, bc=L.BC_PEC)
        a = O.port_uniform(9, y.n_edges)
        b0 = O.port_spmv((c.rows, c.cols, c.row_ptr, c.col_idx, c.val), a)
        y.load(b0, np.zeros(y.n_edges))
        e0 = y.energy()
        y.advance(200)
        out[prec] = (*y.fetch(), y.energy() / e0)
    assert rel_l2(out[4][0], out[8][0]) <= 1e-4
    assert rel_l2(out[4][1], out[8][1]) <= 1e-4
    assert abs(out[4][3] - out[8][3]) <= 1e-5


def test_zero_and_identity_flows():
    y = S.YeeScheme(5, 6, 7, 1, 1, 1, 0.2, bc=L.BC_PEC)
    y.load(np.zeros(y.n_faces), np.zeros(y.n_edges))
    y.advance(10)
    b, e, t = y.fetch()
    assert not b.any() and not e.any() and t == pytest.approx(2.0)
    rng = np.random.default_rng(1)
    b0, e0 = rng.standard_normal(y.n_faces), rng.standard_normal(y.n_edges)
    y.load(b0, e0)
    y.flow_he(0.0)
    y.flow_ha(0.0)
    b, e, _ = y.fetch()
    assert np.array_equal(b, b0) and np.array_equal(e, e0)


@pytest.mark.parametrize("prec", [8, 4])
def test_two_step_sweep_pdl_bitwise(prec):
    """SFEEC_PDL=1: back-to-back two-step sweeps as programmatic dependent
    launches (each waits on griddepcontrol before its first TMA load)."""
    from tests.envutil import layout_env
    dims, d = (45, 19, 70), (1.0, 0.9, 1.1)
    rng = np.random.default_rng(9)
    out = []
    for pdl in ("0", "1"):  # off, on (the default)
        with layout_env(SFEEC_PDL=pdl):
            y = S.YeeScheme(*dims, *d, 0.25, bc=L.BC_PEC, precision=prec)
            y.set_variant(4)
            if not out:
                b0, e0 = rng.standard_normal(y.n_faces), rng.standard_normal(y.n_edges)
            y.load(b0, e0)
            y.advance(23)
            out.append(y.fetch()[:2])
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
