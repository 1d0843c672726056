"""GPU: programmatic dependent launch (PDL) of k_ell / k_sell_pipe changes no
result. SFEEC_PDL is read once per handle (LeapfrogDev::set_pdl)."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from tests.envutil import layout_env

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_programmatic_dependent_launch_bitwise(graphs):
    """The reference arm runs with PDL off (SFEEC_PDL=0), the compared arm
    with the default (on): the same steps, with and without the CUDA-graph
    replay (both arms used to run with PDL on)."""
    rng = np.random.default_rng(11)
    with layout_env(SFEEC_GRAPHS=graphs):
        with layout_env(SFEEC_PDL=0):
            s0 = S.tet_device_scheme(16, 0.1, 3, dt=0.01)
        st = S.make_state(S.Formulation.BE, rng.standard_normal(s0._n2),
                          rng.standard_normal(s0._n1))
        a = s0.advance(st, 70)
        s1 = S.tet_device_scheme(16, 0.1, 3, dt=0.01)
        b = s1.advance(st, 70)
    assert np.array_equal(a.first, b.first) and np.array_equal(a.e, b.e)


def test_pdl_switch_read_once_per_handle():
    """A handle keeps the PDL mode it was created with: flipping SFEEC_PDL
    afterwards changes nothing (graph replay and direct launches agree)."""
    rng = np.random.default_rng(3)
    s = S.tet_device_scheme(12, 0.1, 3, dt=0.01)
    st = S.make_state(S.Formulation.BE, rng.standard_normal(s._n2), rng.standard_normal(s._n1))
    a = s.advance(st, 40)
    with layout_env(SFEEC_PDL=0):
        b = s.advance(st, 40)
    assert np.array_equal(a.first, b.first) and np.array_equal(a.e, b.e)
