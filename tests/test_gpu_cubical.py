"""GPU: cubical (non-lumped) SFEEC -- C, the consistent Q1- M2 and the S(M1)
SPAI of the Q1- M1 on a periodic lattice (the reference's own cubical use,
sfeec_main.cpp cmd_evolve with --lumped off) -- stepped by the device
SplitScheme against the unmodified reference step (oracle/_ref) or the C port."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from oracle import oracle as O
from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu


def tup(a):
    return (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)


@pytest.mark.parametrize("strict", [True, False])
def test_cubical_spai_scheme_matches_reference(strict):
    dims, d = (6, 5, 7), (0.5, 1.0, 0.8)
    c, div = S.yee_operators(*dims, *d, bc=0)
    m1, m2 = S.yee_masses(*dims, *d, bc=0)
    q, rep = S.spai_approximate_inverse(m1, "m1")
    assert rep["fallback_columns"] == 0
    a = O.port_uniform(5, c.cols)
    b0, e0 = O.port_spmv(tup(c), a), O.port_uniform(6, c.cols)
    dt, steps = 0.05, 40
    if O.ref_available():
        ref = O.RefScheme(1, dt, tup(q), tup(c), tup(m2), div=tup(div))
        rb, re_, _, _ = ref.steps(True, b0, e0, steps)
    else:
        port = O.PortScheme(1, dt, tup(q), tup(c), tup(m2), div=tup(div))
        rb, re_, _ = port.steps(b0, e0, steps)
    s = S.SplitScheme(S.SplitKind.Strang, dt, q, c, m2, div=div, warn_cfl=False, strict=strict)
    out = s.advance(S.make_state(S.Formulation.BE, b0, e0), steps)
    if strict:
        assert np.array_equal(out.first, rb) and np.array_equal(out.e, re_)
    else:
        assert rel_l2(out.first, rb) <= 1e-12 and rel_l2(out.e, re_) <= 1e-12
    assert s.gauss_residual(out) <= 1e-12 * np.abs(b0).max()
