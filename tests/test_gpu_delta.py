"""GPU: the sliced SpMV variants against each other and the CSR products:
the TMA-streamed sliced kernel (csrc/stream_spmv.cu, SFEEC_SELL_TMA=1)
against the register-pipelined default, and the compact layouts against the
int32 layouts -- windowed (WUnit in csrc/spmv_kernels.cuh, SFEEC_WIN=1: x
staged in shared memory, 16-bit window indices) and column-delta
(SFEEC_DELTA=1). All three were measured slower than the defaults and are
kept as options.
Every form sums every row in CSR order with the same operations, so the
results are bitwise equal."""
import os
from contextlib import contextmanager

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2301_01753_b200 as S
from paper_2301_01753_b200 import configs
from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu

OPS = ("q_sym", "c", "ct", "m2")


@contextmanager
def layout_env(**env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v


def delta(on: bool):
    return layout_env(SFEEC_WIN=0, SFEEC_DELTA=1 if on else 0)


def win(on: bool):  # the narrow operators too (off by default, measured slower)
    return layout_env(SFEEC_WIN=1 if on else 0, SFEEC_WIN_NARROW=1, SFEEC_DELTA=0)


def csr(a):
    return sp.csr_matrix((a.val, a.col_idx, a.row_ptr), shape=(a.rows, a.cols))


def _check_pair(d1, d0, ops, seed, expect_compact=True, flag="delta"):
    rng = np.random.default_rng(seed)
    for name in OPS:
        a = ops[name]
        x = rng.standard_normal(a.cols)
        y1, y0 = d1.apply(name, x), d0.apply(name, x)
        assert np.array_equal(y1, y0), name
        assert rel_l2(y1, csr(a) @ x) <= 1e-14, name
        i1, i0 = d1.layout_info(name), d0.layout_info(name)
        assert i1["nnz"] == a.nnz() and i1["layout"] == i0["layout"]
        assert i0["delta"] == 0 and i0["win"] == 0
        if i0["layout"] == 0:  # short ragged runs stay CSR in both forms
            assert i1[flag] == 0
            continue
        if expect_compact:
            assert i1[flag] == 1, (name, i1)
            assert i1["stream_bytes"] < i0["stream_bytes"], (name, i1, i0)
            assert i1["full_slices"] <= 0.25 * i1["slices"], (name, i1)


def _advance_pair(d1, d0, n1, n2, steps, seed):
    rng = np.random.default_rng(seed)
    st = S.make_state(S.Formulation.BE, rng.standard_normal(n2), rng.standard_normal(n1))
    x, y = d1.advance(st, steps), d0.advance(st, steps)
    assert np.array_equal(x.first, y.first) and np.array_equal(x.e, y.e)


@pytest.mark.parametrize("n", [5, 12])
def test_tet_device_delta_layout_bitwise_equals_int32_layout(n):
    with delta(True):
        d1 = S.tet_device_scheme(n, 0.12, 9, dt=0.01)
    with delta(False):
        d0 = S.tet_device_scheme(n, 0.12, 9, dt=0.01)
    ops = S.tet_device_operators(n, 0.12, 9)
    _check_pair(d1, d0, ops, n, expect_compact=n >= 12)
    _advance_pair(d1, d0, ops["c"].cols, ops["c"].rows, 25, n)
    # the incidence operators keep the signed (value-free) encoding
    assert d1.layout_info("c")["layout"] == 1 and d1.layout_info("ct")["layout"] == 1


def test_tet_host_built_delta_layout():
    sys_ = configs.tet_system(6, 0.1, 3)
    mk = lambda: S.SplitScheme(S.SplitKind.Strang, 0.01, sys_.q, sys_.c, sys_.m2,
                               warn_cfl=False)
    with delta(True):
        d1 = mk()
    with delta(False):
        d0 = mk()
    ops = {"q_sym": S.symmetric_part(sys_.q), "c": sys_.c, "ct": S.transpose(sys_.c),
           "m2": sys_.m2}
    _check_pair(d1, d0, ops, 6, expect_compact=False)
    _advance_pair(d1, d0, sys_.c.cols, sys_.c.rows, 25, 6)


def test_p2_delta_layout_bitwise_equals_int32_layout():
    with delta(True):
        d1 = S.p2_device_scheme(3, 0.1, 5, dt=0.01)
    with delta(False):
        d0 = S.p2_device_scheme(3, 0.1, 5, dt=0.01)
    ops = S.p2_device_operators(3, 0.1, 5)
    _check_pair(d1, d0, ops, 3, expect_compact=False)
    _advance_pair(d1, d0, ops["c"].cols, ops["c"].rows, 10, 3)


def test_wide_deltas_fall_back_to_int32_columns():
    """Rows whose k-th columns are far apart (random columns) cannot use
    int16 deltas: those slices / ELL groups keep int32 columns; rows with
    local columns next to them still use deltas. Results stay exact."""
    rng = np.random.default_rng(0)
    n1, n2 = 400_000, 120_000

    def rand_op(rows, cols, w, local_rows, signed):
        r = np.repeat(np.arange(rows), w)
        c = np.empty(rows * w, np.int64)
        for i in range(rows):
            if i < local_rows:  # near-diagonal: deltas fit
                lo = min(max(i * cols // rows - 2 * w, 0), cols - 4 * w)
                c[i * w:(i + 1) * w] = lo + np.sort(rng.choice(4 * w, w, replace=False))
            else:  # random columns in the upper half only, so Q_sym and C^T
                # keep local rows in their lower halves
                c[i * w:(i + 1) * w] = cols // 2 + np.sort(rng.choice(cols - cols // 2, w,
                                                                       replace=False))
        v = (rng.choice([-1.0, 1.0], rows * w) if signed else rng.standard_normal(rows * w))
        return S.operator_from_triplets(rows, cols, r, c, v)

    # Q: a symmetric band (|i - j| <= 7) on the lower quarter (32-row slices
    # whose deltas fit), the same band under a random permutation on the
    # upper 3/4 (the same row lengths, columns up to 3e5 apart)
    loc = n1 // 4
    perm = np.concatenate([np.arange(loc), loc + rng.permutation(n1 - loc)])
    rr, cc = [], []
    for lo, hi in ((0, loc), (loc, n1)):
        for d in range(-7, 8):
            i = np.arange(max(lo, lo - d), min(hi, hi - d))
            rr.append(perm[i])
            cc.append(perm[i + d])
    rr, cc = np.concatenate(rr), np.concatenate(cc)
    q = S.operator_from_triplets(n1, n1, rr, cc, rng.standard_normal(rr.size))
    c = rand_op(n2, n1, 3, n2 // 2, True)
    m2 = rand_op(n2, n2, 7, n2 // 2, False)
    mk = lambda: S.SplitScheme(S.SplitKind.Strang, 0.01, q, c, m2, warn_cfl=False)
    with delta(True):
        d1 = mk()
    with delta(False):
        d0 = mk()
    ops = {"q_sym": S.symmetric_part(q), "c": c, "ct": S.transpose(c), "m2": m2}
    _check_pair(d1, d0, ops, 1, expect_compact=False)
    for name in ("q_sym", "c"):  # (C^T: ragged rows; M2: columns within 1.2e5)
        info = d1.layout_info(name)
        assert info["delta"] == 1 and 0 < info["full_slices"] < info["slices"], (name, info)


# ---- windowed layout ---------------------------------------------------------

@pytest.mark.parametrize("n", [6, 16])
def test_tet_device_windowed_layout_bitwise_equals_int32_layout(n):
    with win(True):
        d1 = S.tet_device_scheme(n, 0.12, 9, dt=0.01)
    with win(False):
        d0 = S.tet_device_scheme(n, 0.12, 9, dt=0.01)
    ops = S.tet_device_operators(n, 0.12, 9)
    _check_pair(d1, d0, ops, n, expect_compact=n >= 16, flag="win")
    _advance_pair(d1, d0, ops["c"].cols, ops["c"].rows, 25, n)
    if n >= 16:  # several units per operator, every one of them windowed
        for name in OPS:
            assert d1.layout_info(name)["units"] > 1


def test_tet_host_built_windowed_layout():
    sys_ = configs.tet_system(7, 0.1, 3)
    mk = lambda: S.SplitScheme(S.SplitKind.Strang, 0.01, sys_.q, sys_.c, sys_.m2,
                               warn_cfl=False)
    with win(True):
        d1 = mk()
    with win(False):
        d0 = mk()
    ops = {"q_sym": S.symmetric_part(sys_.q), "c": sys_.c, "ct": S.transpose(sys_.c),
           "m2": sys_.m2}
    _check_pair(d1, d0, ops, 7, expect_compact=False, flag="win")
    _advance_pair(d1, d0, sys_.c.cols, sys_.c.rows, 25, 7)


def test_p2_windowed_layout_bitwise_equals_int32_layout():
    with win(True):
        d1 = S.p2_device_scheme(3, 0.1, 5, dt=0.01)
    with win(False):
        d0 = S.p2_device_scheme(3, 0.1, 5, dt=0.01)
    ops = S.p2_device_operators(3, 0.1, 5)
    _check_pair(d1, d0, ops, 3, expect_compact=False, flag="win")
    _advance_pair(d1, d0, ops["c"].cols, ops["c"].rows, 10, 3)


def test_windows_too_wide_fall_back():
    """Rows with random columns over 4e5 ids: no unit size gives windows of
    at most 14336 values, so the operator keeps the int32 layout; an odd
    number of columns exercises the odd-tail copy of the window staging."""
    rng = np.random.default_rng(2)
    n1, n2 = 400_001, 3_001
    r = np.repeat(np.arange(n2), 12)  # 64-row units: 768 blocks > 448
    cwide = np.concatenate([np.sort(rng.choice(n1, 12, replace=False)) for _ in range(n2)])
    c = S.operator_from_triplets(n2, n1, r, cwide, rng.choice([-1.0, 1.0], r.size))
    q = S.scaled_identity(n1, 2.0)
    m2 = S.scaled_identity(n2, 0.5)
    with win(True):
        d1 = S.SplitScheme(S.SplitKind.Strang, 0.01, q, c, m2, warn_cfl=False)
    x = rng.standard_normal(n1)
    assert rel_l2(d1.apply("c", x), csr(c) @ x) <= 1e-14
    assert d1.layout_info("c")["win"] == 0
    # a narrow band with an odd column count is windowed, tail included
    nb = 4_097
    rb = np.repeat(np.arange(nb), 3)
    cb = np.clip(np.repeat(np.arange(nb), 3) + np.tile([-1, 0, 1], nb), 0, nb - 1)
    band = S.operator_from_triplets(nb, nb, rb, cb, rng.standard_normal(rb.size))
    with win(True):
        d2 = S.SplitScheme(S.SplitKind.Strang, 0.01, S.scaled_identity(nb, 1.0), band,
                           S.scaled_identity(nb, 1.0), warn_cfl=False)
    xb = rng.standard_normal(nb)
    assert d2.layout_info("c")["win"] == 1
    assert np.array_equal(d2.apply("c", xb), d2.apply("c", xb))
    assert rel_l2(d2.apply("c", xb), csr(band) @ xb) <= 1e-14


def test_default_layouts_window_only_the_wide_operators():
    with layout_env(SFEEC_WIN=1, SFEEC_WIN_NARROW=0, SFEEC_DELTA=0):
        d = S.tet_device_scheme(16, 0.12, 9, dt=0.01)
    assert d.layout_info("q_sym")["win"] == 1
    for name in ("c", "ct", "m2"):
        info = d.layout_info(name)
        assert info["win"] == 0 and info["ell"] == 1, (name, info)


# ---- TMA-streamed sliced kernel ------------------------------------------------

def _wide_band_scheme(n1=20_000, half=50, seed=3):
    """Q_sym: a symmetric band of 101 entries per row (sliced, 7 stages per
    slice in the TMA-streamed kernel: the config-4 shape)."""
    rng = np.random.default_rng(seed)
    rr, cc = [], []
    for d in range(-half, half + 1):
        i = np.arange(max(0, -d), min(n1, n1 - d))
        rr.append(i)
        cc.append(i + d)
    rr, cc = np.concatenate(rr), np.concatenate(cc)
    q = S.operator_from_triplets(n1, n1, rr, cc, rng.standard_normal(rr.size))
    n2 = n1 + 7
    r = np.repeat(np.arange(n2), 3)
    c = S.operator_from_triplets(n2, n1, r, (r * 7 + np.tile([0, 1, 5], n2)) % n1,
                                 rng.choice([-1.0, 1.0], r.size))
    m2 = S.scaled_identity(n2, 0.5)
    ops = {"q_sym": S.symmetric_part(q), "c": c, "ct": S.transpose(c), "m2": m2}
    return (lambda: S.SplitScheme(S.SplitKind.Strang, 0.01, q, c, m2, warn_cfl=False)), ops


@pytest.mark.parametrize("kind,n", [("tet", 12), ("tet", 20), ("wide", 0)])
def test_sell_tma_bitwise_equals_register_pipelined(kind, n):
    if kind == "tet":
        mk = lambda: S.tet_device_scheme(n, 0.12, 9, dt=0.01)
        ops = S.tet_device_operators(n, 0.12, 9)
    else:
        mk, ops = _wide_band_scheme()
    with layout_env(SFEEC_SELL_TMA=1):
        d1 = mk()
    with layout_env(SFEEC_SELL_TMA=0):
        d0 = mk()
    rng = np.random.default_rng(n)
    for name in OPS:
        x = rng.standard_normal(ops[name].cols)
        with layout_env(SFEEC_SELL_TMA=1):
            y1 = d1.apply(name, x)
        with layout_env(SFEEC_SELL_TMA=0):
            y0 = d0.apply(name, x)
        assert np.array_equal(y1, y0), name
        assert rel_l2(y1, csr(ops[name]) @ x) <= 1e-14, name
    if n >= 20 or kind == "wide":  # (small tet meshes keep Q in CSR: ragged runs)
        assert d1.layout_info("q_sym")["layout"] == 2 and d1.layout_info("q_sym")["ell"] == 0
    st = S.make_state(S.Formulation.BE, rng.standard_normal(ops["c"].rows),
                      rng.standard_normal(ops["c"].cols))
    with layout_env(SFEEC_SELL_TMA=1):
        x1 = d1.advance(st, 12)
    with layout_env(SFEEC_SELL_TMA=0):
        x0 = d0.advance(st, 12)
    assert np.array_equal(x1.first, x0.first) and np.array_equal(x1.e, x0.e)
