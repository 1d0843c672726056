"""CPU: pin the oracle (plain-C port) against the reference's golden fixtures,
and against the reference library itself when it is built (oracle/_ref)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import rel_l2


def _ops(g):
    n1, n2 = int(g["n1"]), int(g["n2"])
    q = (n1, n1, g["q_rp"], g["q_ci"], g["q_va"])
    c = (n2, n1, g["c_rp"], g["c_ci"], g["c_va"])
    m2 = (n2, n2, g["m2_rp"], g["m2_ci"], g["m2_va"])
    return q, c, m2


def test_port_symmetric_part_matches_reference_bitwise(golden):
    g = golden("scheme.npz")
    q, _, _ = _ops(g)
    qs = O.port_symmetric_part(q)
    assert np.array_equal(qs[2], g["qsym_rp"])
    assert np.array_equal(qs[3], g["qsym_ci"])
    assert np.array_equal(qs[4], g["qsym_va"])


@pytest.mark.parametrize("strang", [1, 0])
@pytest.mark.parametrize("be", [1, 0])
def test_port_steps_match_reference_bitwise(golden, strang, be):
    g = golden("scheme.npz")
    q, c, m2 = _ops(g)
    key = f"s{strang}b{be}"
    s = O.PortScheme(strang, 0.05, q, c, m2, be=bool(be))
    first0 = g["b0"] if be else g["a0"]
    f1, e1, hist = s.steps(first0, g["e0"], 20, energy=True)
    assert np.array_equal(f1, g[f"{key}_first"])
    assert np.array_equal(e1, g[f"{key}_e"])
    assert np.array_equal(hist, g[f"{key}_energy"])
    assert s.energy(first0, g["e0"]) == g[f"{key}_energy0"]
    fh, eh = s.flow_he(first0, g["e0"], 0.34)
    assert np.array_equal(fh, g[f"{key}_flowhe_first"]) and np.array_equal(eh, g[f"{key}_flowhe_e"])
    fa, ea = s.flow_ha(first0, g["e0"], 0.7)
    assert np.array_equal(fa, g[f"{key}_flowha_first"]) and np.array_equal(ea, g[f"{key}_flowha_e"])
    assert s.cfl() == g[f"{key}_cfl"]


def test_port_yee_fdtd_matches_reference_bitwise(golden):
    g = golden("yee.npz")
    nx, ny, nz = (int(v) for v in g["dims"])
    d, dt, steps = g["d"], float(g["dt"]), int(g["steps"])
    b = O.port_yee_advance_b(nx, ny, nz, d, g["e0"], g["bgrid0"], 0.5 * dt)
    e, b = O.port_yee_step(nx, ny, nz, d, g["e0"], b, dt, steps)
    assert np.array_equal(e, g["e_fdtd"])
    assert np.array_equal(b, g["b_fdtd"])


def test_lumped_sfeec_equals_fdtd_reference_contract(golden):
    """test_yee.cpp:157-163 / SPEC.md: lumped SFEEC == FDTD to <= 1e-12."""
    g = golden("yee.npz")
    d = g["d"]
    dv = d[0] * d[1] * d[2]
    assert np.max(np.abs(g["e_sfeec"] - g["e_fdtd"])) <= 1e-12
    assert np.max(np.abs(dv * g["b_sfeec_staggered"] - g["b_fdtd"])) <= 1e-12


def test_port_from_triplets_matches_reference(golden):
    g = golden("triplets.npz")
    m = O.port_from_triplets(7, 5, g["r"], g["c"], g["v"])
    assert np.array_equal(m[2], g["rp"]) and np.array_equal(m[3], g["ci"])
    assert np.array_equal(m[4], g["va"])


def test_port_uniform_is_splitmix64():
    # core.hpp:44-63 first outputs for seed 0 (splitmix64 reference values)
    s = O.port_uniform(0, 2, 0.0, 1.0)
    z = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]
    assert np.array_equal(s, [(v >> 11) * 2.0 ** -53 for v in z])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_port_equals_live_reference_on_fresh_inputs():
    """Fresh seeded operators, not in the fixtures: port and reference bitwise."""
    rng = np.random.default_rng(42)
    from tests.golden.make_golden import synthetic_ops
    q, c, m2, cs = synthetic_ops(n=2, seed=5)
    a0 = rng.standard_normal(c[1])
    e0 = rng.standard_normal(c[1])
    for strang in (0, 1):
        r = O.RefScheme(strang, 0.07, q, c, m2, eps0=2.5, mu0=0.4)
        p = O.PortScheme(strang, 0.07, q, c, m2, eps0=2.5, mu0=0.4, be=True)
        b0 = cs @ a0
        rf, re, _, rh = r.steps(1, b0, e0, 13, energy=True)
        pf, pe, ph = p.steps(b0, e0, 13, energy=True)
        assert np.array_equal(rf, pf) and np.array_equal(re, pe) and np.array_equal(rh, ph)
        assert r.cfl() == p.cfl()
    assert rel_l2(O.port_spmv(q, e0), O.ref_spmv(q, e0)) == 0.0
