"""GPU: the column-delta layouts (DSlice in csrc/spmv_kernels.cuh; the
production default) against the int32-column layouts (SFEEC_DELTA=0) and
the CSR products. Both forms sum every row in CSR order with the same
operations, so the results are bitwise equal; the delta form streams fewer
bytes. Slices whose deltas leave the int16 range keep int32 columns."""
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
def delta(on: bool):
    old = os.environ.get("SFEEC_DELTA")
    os.environ["SFEEC_DELTA"] = "1" if on else "0"
    try:
        yield
    finally:
        if old is None:
            os.environ.pop("SFEEC_DELTA")
        else:
            os.environ["SFEEC_DELTA"] = old


def csr(a):
    return sp.csr_matrix((a.val, a.col_idx, a.row_ptr), shape=(a.rows, a.cols))


def _check_pair(d1, d0, ops, seed, expect_compact=True):
    rng = np.random.default_rng(seed)
    for name in OPS:
        a = ops[name]
        x = rng.standard_normal(a.cols)
        y1, y0 = d1.apply(name, x), d0.apply(name, x)
        assert np.array_equal(y1, y0), name
        assert rel_l2(y1, csr(a) @ x) <= 1e-14, name
        i1, i0 = d1.layout_info(name), d0.layout_info(name)
        assert i1["nnz"] == a.nnz() and i1["layout"] == i0["layout"]
        assert i0["delta"] == 0
        if i0["layout"] == 0:  # short ragged runs stay CSR in both forms
            assert i1["delta"] == 0
            continue
        if expect_compact:
            assert i1["delta"] == 1, (name, i1)
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
