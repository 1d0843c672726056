"""GPU: the Kuhn-lattice step (csrc/lattice.cu) against the
sliced / ELL step on the same device-assembled operators, and the handle's
state bookkeeping between the lattice state and the DOF vectors."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu


def _pair(n, jit=0.1, seed=3, dt=0.01, kind=S.SplitKind.Strang):
    lat = S.tet_device_scheme(n, jit, seed, dt=dt, kind=kind, layout="lattice")
    sell = S.tet_device_scheme(n, jit, seed, dt=dt, kind=kind, layout="sell")
    return lat, sell


@pytest.mark.parametrize("n", [1, 2, 3, 12, 33, 40])
@pytest.mark.parametrize("kind", [S.SplitKind.Strang, S.SplitKind.LieTrotter])
def test_lattice_step_matches_sliced_step(n, kind):
    """33 and 40 vertices per row span two 32-vertex x-blocks (rows at the
    block edge sum in another order); 3 has no interior vertex at all"""
    lat, sell = _pair(n, kind=kind)
    rng = np.random.default_rng(n)
    st = S.make_state(S.Formulation.BE, rng.standard_normal(lat._n2),
                      rng.standard_normal(lat._n1))
    a, b = lat.advance(st, 37), sell.advance(st, 37)
    assert rel_l2(a.first, b.first) <= 1e-13 and rel_l2(a.e, b.e) <= 1e-13
    assert lat.energy(a) == pytest.approx(sell.energy(b), rel=1e-13)
    assert a.time == b.time


def test_lattice_interior_rows_sum_in_csr_order():
    """n = 8: one x-block per row, so every row sums in CSR order and the
    lattice step is bitwise the sliced step"""
    lat, sell = _pair(8)
    rng = np.random.default_rng(1)
    st = S.make_state(S.Formulation.BE, rng.standard_normal(lat._n2),
                      rng.standard_normal(lat._n1))
    a, b = lat.advance(st, 20), sell.advance(st, 20)
    assert np.allclose(a.first, b.first, rtol=0, atol=1e-14 * np.abs(b.first).max())
    assert np.allclose(a.e, b.e, rtol=0, atol=1e-14 * np.abs(b.e).max())


def test_lattice_state_sync_between_calls():
    """advance, diagnostics and reloads interleave: the lattice state is
    gathered when the DOF vectors are read and re-scattered after a load"""
    lat, _ = _pair(10)
    rng = np.random.default_rng(2)
    st = S.make_state(S.Formulation.BE, rng.standard_normal(lat._n2),
                      rng.standard_normal(lat._n1))
    # two advance() calls (each opens and closes with a half-kick)
    whole = lat.advance(lat.advance(st, 10), 20)
    lat.load(st)
    lat.advance_resident(10)
    e10 = lat.energy_resident()       # gathers, lattice stays valid
    mid = lat.fetch()                 # gathers
    lat.advance_resident(20)
    two = lat.fetch()
    assert np.array_equal(two.first, whole.first) and np.array_equal(two.e, whole.e)
    assert e10 == pytest.approx(lat.energy(mid), rel=0)
    # a reload after lattice steps replaces the lattice state
    lat.advance_resident(3)
    again = lat.advance(lat.advance(st, 10), 20)
    assert np.array_equal(again.first, whole.first)
    # half-flows through the ABI run on the DOF vectors of the lattice state
    lat.load(st)
    lat.advance_resident(5)
    lat.flow_he_resident(0.0)  # zero-length flow: the state is unchanged
    five = lat.fetch()
    ref = lat.advance(st, 5)
    assert np.array_equal(five.first, ref.first) and np.array_equal(five.e, ref.e)


def test_lattice_kernel_timing_reports_lattice_bytes():
    lat, sell = _pair(16)
    rng = np.random.default_rng(0)
    st = S.make_state(S.Formulation.BE, rng.standard_normal(lat._n2),
                      rng.standard_normal(lat._n1))
    lat.load(st)
    sell.load(st)
    out = {}
    for name, s in (("lat", lat), ("sell", sell)):
        s.kernel_timing(True)
        s.advance_resident(8)
        out[name] = s.kernel_timing(False)
    V = 17 ** 3
    assert out["lat"]["K-Q"]["bytes_per_launch"] == 8.0 * (61 * V + 7 * V + lat._n1)
    assert out["lat"]["K-M2"]["bytes_per_launch"] == 8.0 * (48 * V + 12 * V + lat._n2)
    for k in ("K-Q", "K-Cb", "K-CTe", "K-M2"):
        assert out["lat"][k]["launches"] == out["sell"][k]["launches"] > 0
        # the lattice moves fewer bytes than the sliced layouts' accounting
        assert out["lat"][k]["bytes_per_launch"] < out["sell"][k]["bytes_per_launch"]
