"""GPU: the tet system assembled on the device (tet_device.cu) equals the
host builders bit for bit (which equal the numpy construction oracle), and a
device-assembled scheme steps like the host-built one."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200 import configs
from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu


def same(a, b):
    return (a.rows == b.rows and a.cols == b.cols and np.array_equal(a.row_ptr, b.row_ptr)
            and np.array_equal(a.col_idx, b.col_idx) and np.array_equal(a.val, b.val))


@pytest.mark.parametrize("n,jit,seed", [(4, 0.1, 7), (9, 0.15, 3)])
def test_device_assembly_bitwise_equals_host(n, jit, seed):
    dev = S.tet_device_operators(n, jit, seed)
    mesh = S.TetMesh(n, jit, seed)
    assert same(dev["c"], mesh.curl())
    assert same(dev["m2"], mesh.mass2())
    assert same(dev["d"], mesh.div())
    assert same(dev["ct"], S.transpose(mesh.curl()))
    q, rep = S.spai_approximate_inverse(mesh.mass1(), "m1")
    assert rep["fallback_columns"] == 0
    assert same(dev["q_sym"], S.symmetric_part(q))


@pytest.mark.parametrize("layout", ["host", "sell", "device", "lattice"])
def test_device_scheme_matches_host_scheme(layout):
    n, jit, seed = 8, 0.1, 5
    sys_ = configs.tet_system(n, jit, seed)
    b0, e0, a = configs.initial_gaussian(sys_, seed=4)
    host = S.SplitScheme(S.SplitKind.Strang, 0.02, sys_.q, sys_.c, sys_.m2, div=sys_.d,
                         warn_cfl=False)
    dev = S.tet_device_scheme(n, jit, seed, dt=0.02, layout=layout)
    assert np.array_equal(dev.apply("c", a), b0) or np.allclose(dev.apply("c", a), b0, rtol=0,
                                                                  atol=1e-15)
    assert dev.cfl_number() == pytest.approx(host.cfl_number(), rel=1e-12)
    st = S.make_state(S.Formulation.BE, b0, e0)
    x, y = host.advance(st, 30), dev.advance(st, 30)
    if layout in ("host", "sell", "device"):  # same operators, same kernels (n < 48): bitwise
        assert np.array_equal(x.first, y.first) and np.array_equal(x.e, y.e)
    else:  # the lattice step: rows at the x-block edges sum in another order
        assert rel_l2(y.first, x.first) <= 1e-13 and rel_l2(y.e, x.e) <= 1e-13
    assert dev.gauss_residual(y) <= 1e-12 * np.abs(b0).max()


@pytest.mark.parametrize("layout", ["device", "host"])
@pytest.mark.parametrize("n", [5, 12])
def test_device_layouts_apply_the_csr_operators(n, layout):
    """Every operator of the device handle equals its CSR product."""
    import scipy.sparse as sp
    dev = S.tet_device_scheme(n, 0.12, 9, layout=layout)
    ops = S.tet_device_operators(n, 0.12, 9)
    rng = np.random.default_rng(n)
    for name, key in (("q_sym", "q_sym"), ("c", "c"), ("ct", "ct"), ("m2", "m2")):
        a = ops[key]
        m = sp.csr_matrix((a.val, a.col_idx, a.row_ptr), shape=(a.rows, a.cols))
        x = rng.standard_normal(a.cols)
        assert rel_l2(dev.apply(name, x), m @ x) <= 1e-14, name
