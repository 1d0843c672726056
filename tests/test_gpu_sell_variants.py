"""GPU: the sliced SpMV variants selectable by SFEEC_SELL_VARIANT (register
pipelined k_sell_pipe = 9..13, + L2 bulk prefetch k_sell_pf = 14..16) give
bitwise the same rows (same per-row FMA order) on the tet operators."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from tests.test_gpu_delta import layout_env

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", [14, 15, 16])
def test_prefetch_variants_bitwise(variant):
    s = S.tet_device_scheme(16, 0.1, 3, dt=0.01)
    rng = np.random.default_rng(variant)
    x = rng.standard_normal(s._n1)
    ref = s.apply("q_sym", x)
    with layout_env(SFEEC_SELL_VARIANT=variant):
        out = s.apply("q_sym", x)
        st = S.make_state(S.Formulation.BE, rng.standard_normal(s._n2), rng.standard_normal(s._n1))
        a = s.advance(st, 9)
    assert np.array_equal(out, ref)
    b = s.advance(st, 9)
    assert np.array_equal(a.first, b.first) and np.array_equal(a.e, b.e)


def test_prefetch_wide_rows_bitwise():
    """config 4's S(M1^2) Q: ~300 entries per row, in-slice prefetches"""
    s = S.p2_device_scheme(3, 0.1, 2, dt=0.005)
    x = np.random.default_rng(1).standard_normal(s._n1)
    ref = s.apply("q_sym", x)
    with layout_env(SFEEC_SELL_VARIANT=14):
        out = s.apply("q_sym", x)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("n", [16, 24])
def test_alternating_row_order_bitwise(n):
    """SFEEC_ALT_DIR=1 runs M2 and Q in descending row order: same rows."""
    s = S.tet_device_scheme(n, 0.1, 3, dt=0.01)
    rng = np.random.default_rng(n)
    st = S.make_state(S.Formulation.BE, rng.standard_normal(s._n2), rng.standard_normal(s._n1))
    a = s.advance(st, 40)
    with layout_env(SFEEC_ALT_DIR=1):
        b = s.advance(st, 40)
    assert np.array_equal(a.first, b.first) and np.array_equal(a.e, b.e)


@pytest.mark.parametrize("pf", [1, 2, 4, 6])
def test_l2_prefetch_size_hint_bitwise(pf):
    """SFEEC_L2PF=1/2 adds .L2::128B/.L2::256B to the operator streams of
    k_ell and k_sell_pipe: same loads, same rows, same steps."""
    s = S.tet_device_scheme(16, 0.1, 3, dt=0.01)
    rng = np.random.default_rng(pf)
    x, z = rng.standard_normal(s._n1), rng.standard_normal(s._n2)
    ref = [s.apply(w, v) for w, v in (("q_sym", x), ("c", x), ("ct", z), ("m2", z))]
    st = S.make_state(S.Formulation.BE, rng.standard_normal(s._n2), rng.standard_normal(s._n1))
    a = s.advance(st, 9)
    with layout_env(SFEEC_L2PF=pf):
        out = [s.apply(w, v) for w, v in (("q_sym", x), ("c", x), ("ct", z), ("m2", z))]
        b = s.advance(st, 9)
    for o, r in zip(out, ref):
        assert np.array_equal(o, r)
    assert np.array_equal(a.first, b.first) and np.array_equal(a.e, b.e)


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_programmatic_dependent_launch_bitwise(graphs):
    """SFEEC_PDL=1 launches k_ell / k_sell_pipe as programmatic dependents
    (prologue and operator loads overlap the previous kernel's tail, data
    reads after griddepcontrol.wait): the same steps, with and without the
    CUDA-graph replay."""
    rng = np.random.default_rng(11)
    with layout_env(SFEEC_GRAPHS=graphs):
        s = S.tet_device_scheme(16, 0.1, 3, dt=0.01)
        st = S.make_state(S.Formulation.BE, rng.standard_normal(s._n2), rng.standard_normal(s._n1))
        a = s.advance(st, 70)
        with layout_env(SFEEC_PDL=1):
            s2 = S.tet_device_scheme(16, 0.1, 3, dt=0.01)
            b = s2.advance(st, 70)
    assert np.array_equal(a.first, b.first) and np.array_equal(a.e, b.e)
