"""GPU: the table-driven Kuhn-lattice step (csrc/table_lattice.cu, DESIGN.md
3.6). On the first-order system it must reproduce the sliced step and the
compile-time-unrolled lattice (csrc/lattice.cu); on the second-order system
(config 4's layout) the sliced step on the same device-built operators."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu


def _state(s, seed):
    rng = np.random.default_rng(seed)
    return S.make_state(S.Formulation.BE, rng.standard_normal(s._n2), rng.standard_normal(s._n1))


@pytest.mark.parametrize("n", [4, 7, 12, 33])
@pytest.mark.parametrize("kind", [S.SplitKind.Strang, S.SplitKind.LieTrotter])
def test_first_order_table_step_matches_sliced_and_unrolled_lattice(n, kind):
    tab = S.tet_device_scheme(n, 0.1, 3, dt=0.01, kind=kind, layout="table")
    sell = S.tet_device_scheme(n, 0.1, 3, dt=0.01, kind=kind, layout="sell")
    lat = S.tet_device_scheme(n, 0.1, 3, dt=0.01, kind=kind, layout="lattice")
    st = _state(tab, n)
    a, b, c = tab.advance(st, 37), sell.advance(st, 37), lat.advance(st, 37)
    assert rel_l2(a.first, b.first) <= 1e-13 and rel_l2(a.e, b.e) <= 1e-13
    assert rel_l2(a.first, c.first) <= 1e-13 and rel_l2(a.e, c.e) <= 1e-13
    assert tab.energy(a) == pytest.approx(sell.energy(b), rel=1e-13)
    assert a.time == b.time


def test_first_order_table_rows_sum_in_csr_order():
    """n = 8: one x-block per row, so the slot order (the CSR order of an
    interior row) is every row's CSR order: bitwise-level agreement"""
    tab = S.tet_device_scheme(8, 0.1, 3, dt=0.01, layout="table")
    sell = S.tet_device_scheme(8, 0.1, 3, dt=0.01, layout="sell")
    st = _state(tab, 1)
    a, b = tab.advance(st, 20), sell.advance(st, 20)
    assert np.allclose(a.first, b.first, rtol=0, atol=1e-14 * np.abs(b.first).max())
    assert np.allclose(a.e, b.e, rtol=0, atol=1e-14 * np.abs(b.e).max())


def test_table_lattice_needs_an_interior_vertex():
    with pytest.raises(S.InvalidParameter):
        S.tet_device_scheme(3, 0.1, 3, dt=0.01, layout="table")


@pytest.mark.parametrize("n,kind", [(6, S.SplitKind.Strang), (8, S.SplitKind.Strang),
                                    (6, S.SplitKind.LieTrotter)])
def test_second_order_table_step_matches_sliced(n, kind):
    """P2-, S(M1^2): 38 + 54 DOF types per vertex, two halo layers"""
    tab = S.p2_device_scheme(n, 0.1, 5, dt=2e-3, kind=kind, layout="lattice")
    sell = S.p2_device_scheme(n, 0.1, 5, dt=2e-3, kind=kind, layout="sell")
    st = _state(tab, n)
    a, b = tab.advance(st, 25), sell.advance(st, 25)
    assert rel_l2(a.first, b.first) <= 1e-12 and rel_l2(a.e, b.e) <= 1e-12
    assert tab.energy(a) == pytest.approx(sell.energy(b), rel=1e-12)
    # (a random b is not divergence-free: the residual is only preserved)
    assert tab.gauss_residual(a) == pytest.approx(sell.gauss_residual(st), rel=1e-9)


def test_second_order_state_sync_and_timing_bytes():
    tab = S.p2_device_scheme(6, 0.1, 5, dt=2e-3, layout="lattice")
    st = _state(tab, 2)
    whole = tab.advance(tab.advance(st, 4), 6)
    tab.load(st)
    tab.advance_resident(4)
    e4 = tab.energy_resident()
    mid = tab.fetch()
    tab.advance_resident(6)
    two = tab.fetch()
    assert np.array_equal(two.first, whole.first) and np.array_equal(two.e, whole.e)
    assert e4 == pytest.approx(tab.energy(mid), rel=0)
    tab.kernel_timing(True)
    tab.advance_resident(3)
    t = tab.kernel_timing(False)
    assert t["K-Q"]["launches"] > 0 and t["K-Q"]["bytes_per_launch"] > 0
