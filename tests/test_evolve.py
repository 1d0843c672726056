"""The evolve driver (reference tools/sfeec_main.cpp:151-215): initial state
from one Rng stream, the CSV history format and checkpoints (CPU); the device
history against the reference SplitScheme stepped the same way (GPU)."""
import numpy as np
import pytest

import paper_2301_01753_b200 as S
from oracle import oracle as O
from paper_2301_01753_b200 import configs, evolve


def test_initial_state_is_one_rng_stream():
    sys_ = configs.tet_system(3, 0.1, seed=2)
    st = evolve.evolve_initial_state(sys_.c, 99)
    ae = O.port_uniform(99, 2 * sys_.n1)
    np.testing.assert_array_equal(st.e, ae[sys_.n1:])
    np.testing.assert_array_equal(st.first, O.port_spmv(tup(sys_.c), ae[:sys_.n1]))
    ae_state = evolve.evolve_initial_state(sys_.c, 99, S.Formulation.AE)
    np.testing.assert_array_equal(ae_state.first, ae[:sys_.n1])


def tup(a):
    return (a.rows, a.cols, a.row_ptr, a.col_idx, a.val)


def test_history_format_and_checkpoint(tmp_path):
    text = "step,time,energy,gauss_residual\n" + evolve._row(0, 0.0, 1.5, 0.0) + \
        evolve._row(7, 0.07000000000000001, 1.4999999999999998, 3e-17)
    assert text.splitlines()[2] == "7,0.070000000000000007,1.4999999999999998,3.0000000000000001e-17"
    h = evolve.read_history(text)
    assert h.shape == (2, 4) and h[1, 0] == 7
    st = S.make_state(S.Formulation.BE, np.arange(5.0), np.ones(3), 0.25)
    evolve.save_checkpoint(str(tmp_path / "ck.npz"), st)
    back = evolve.load_checkpoint(str(tmp_path / "ck.npz"))
    assert back.formulation == st.formulation and back.time == st.time
    np.testing.assert_array_equal(back.first, st.first)
    np.testing.assert_array_equal(back.e, st.e)


@pytest.mark.gpu
@pytest.mark.parametrize("strict", [True, False])
def test_device_history_matches_reference_evolve(strict):
    sys_ = configs.tet_system(4, 0.1, seed=3)
    dt, steps, every = 0.01, 23, 5
    st = evolve.evolve_initial_state(sys_.c, 7)
    scheme = S.SplitScheme(S.SplitKind.Strang, dt, sys_.q, sys_.c, sys_.m2, div=sys_.d,
                           warn_cfl=False, strict=strict)
    got = evolve.read_history(evolve.evolve(scheme, st, steps, every))
    # the reference loop of cmd_evolve on the unmodified SplitScheme (oracle/_ref),
    # or the C restatement when _ref is absent
    rows = []
    if O.ref_available():
        ref = O.RefScheme(1, dt, tup(sys_.q), tup(sys_.c), tup(sys_.m2), div=tup(sys_.d))
        b, e, t = st.first, st.e, 0.0
        rows.append((0, t, ref.energy(True, b, e), ref.gauss(b, e)))
        for s in range(1, steps + 1):
            b, e, t, _ = ref.steps(True, b, e, 1, time=t)
            if s % every == 0 or s == steps:
                rows.append((s, t, ref.energy(True, b, e), ref.gauss(b, e)))
    else:
        port = O.PortScheme(1, dt, tup(sys_.q), tup(sys_.c), tup(sys_.m2), div=tup(sys_.d))
        b, e, t = st.first, st.e, 0.0
        rows.append((0, t, port.energy(b, e), port.gauss(b)))
        for s in range(1, steps + 1):
            b, e, _ = port.steps(b, e, 1)
            t = t + dt
            if s % every == 0 or s == steps:
                rows.append((s, t, port.energy(b, e), port.gauss(b)))
    want = np.array(rows)
    assert got.shape == want.shape
    np.testing.assert_array_equal(got[:, :2], want[:, :2])       # steps and times exact
    np.testing.assert_allclose(got[:, 2], want[:, 2], rtol=1e-12)  # energy
    assert np.abs(got[:, 3] - want[:, 3]).max() <= 1e-13 * np.abs(st.first).max()
    fin = scheme.fetch()
    assert fin.time == want[-1, 1]


@pytest.mark.gpu
@pytest.mark.parametrize("strict", [True, False])
def test_curl_of_curl_matches_sequential_products(strict):
    """apply_curl_of_curl (operators.cpp:268-290) = Q C^T M2 C a by sequential
    CSR products (the oracle's spmv); strict kernels bitwise."""
    sys_ = configs.tet_system(4, 0.1, seed=8)
    scheme = S.SplitScheme(S.SplitKind.Strang, 0.01, sys_.q, sys_.c, sys_.m2, warn_cfl=False,
                           strict=strict)
    a = np.random.default_rng(3).standard_normal(sys_.n1)
    qs = tup(S.symmetric_part(sys_.q))
    want = O.port_spmv(qs, O.port_spmv(tup(S.transpose(sys_.c)),
                                       O.port_spmv(tup(sys_.m2), O.port_spmv(tup(sys_.c), a))))
    got = scheme.curl_of_curl(a)
    if strict:
        np.testing.assert_array_equal(got, want)
    else:
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)
