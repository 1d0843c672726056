"""TEST INFRASTRUCTURE ONLY -- the CPU checkers for the B200 leapfrog.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module, and only as the checker or the
reference CPU arm -- never as the product path.

Two checkers, loaded with ctypes:
  * ref   oracle/_ref/libsfeec_ref.so: the UNMODIFIED reference sources
          (/root/reference/proj/src/{sparse,dynamics,yee,mesh_cubical}.cpp)
          compiled by oracle/Makefile with the reference flags, behind the
          extern "C" glue of oracle/ref_shim.cpp.
  * port  oracle/_build/libsfeec_oracle.so: the plain-C restatement
          (oracle/sfeec_oracle.c) -- bitwise equal to `ref` on the same
          inputs; pinned against `ref` and against tests/golden/*.npz.

  * refsetup  oracle/_ref/libsfeec_ref_setup.so: the WHOLE unmodified
          reference library (setup code included: form_space, operators,
          spai) over the Eigen-subset stand-in oracle/eigen_shim, behind
          oracle/ref_shim_setup.cpp: the reference's own make_pattern,
          spai_approximate_inverse, mass_matrix and derivative_matrix.

Parity status: the step arithmetic, the sparse utilities, the Yee FDTD and
the periodic cubical curl are pinned by the reference itself (bitwise). The
3-D tet construction has no reference counterpart; it is pinned by the
invariants of SURVEY.md Appendix C (see tests/test_tetmesh.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(HERE, "_ref", "libsfeec_ref.so")
PORT_PATH = os.path.join(HERE, "_build", "libsfeec_oracle.so")

_PD = C.POINTER(C.c_double)
_PI = C.POINTER(C.c_int)
_PI64 = C.POINTER(C.c_int64)
_PI32 = C.POINTER(C.c_int32)


def build(with_ref: bool = True) -> None:
    """Compile the checkers (oracle/Makefile). The ref build needs /root/reference."""
    targets = ["_build/libsfeec_oracle.so"]
    if with_ref and os.path.isdir("/root/reference/proj/src"):
        targets += ["ref", "refsetup"]
    subprocess.run(["make", "-s", *targets], cwd=HERE, check=True)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(_PD)


# --------------------------------------------------------------------------
# reference library
# --------------------------------------------------------------------------
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref_lib():
    global _ref
    if _ref is None:
        l = C.CDLL(REF_PATH)
        l.sfeec_ref_last_error.restype = C.c_char_p
        l.sfeec_ref_scheme_create.restype = C.c_void_p
        l.sfeec_ref_scheme_create.argtypes = [
            C.c_int, C.c_double, C.c_int, _PI, _PI, _PD, C.c_int, C.c_int, _PI, _PI, _PD, _PI,
            _PI, _PD, C.c_double, C.c_double, C.c_int, _PI, _PI, _PD, C.c_int]
        l.sfeec_ref_scheme_destroy.argtypes = [C.c_void_p]
        l.sfeec_ref_scheme_qsym_nnz.argtypes = [C.c_void_p]
        l.sfeec_ref_scheme_qsym.argtypes = [C.c_void_p, _PI, _PI, _PD]
        l.sfeec_ref_scheme_curl_t.argtypes = [C.c_void_p, _PI, _PI, _PD]
        l.sfeec_ref_scheme_steps.argtypes = [C.c_void_p, C.c_int, _PD, C.c_int, _PD, C.c_int,
                                             _PD, C.c_int, _PD, _PD]
        l.sfeec_ref_scheme_flow.argtypes = [C.c_void_p, C.c_int, C.c_int, _PD, C.c_int, _PD,
                                            C.c_int, C.c_double]
        l.sfeec_ref_scheme_energy.argtypes = [C.c_void_p, C.c_int, _PD, C.c_int, _PD, C.c_int,
                                              _PD]
        l.sfeec_ref_scheme_gauss.argtypes = l.sfeec_ref_scheme_energy.argtypes
        l.sfeec_ref_scheme_cfl.argtypes = [C.c_void_p, _PD]
        l.sfeec_ref_spmv.argtypes = [C.c_int, C.c_int, _PI, _PI, _PD, _PD, _PD]
        l.sfeec_ref_from_triplets.argtypes = [C.c_int, C.c_int, C.c_int, _PI, _PI, _PD, _PI,
                                              _PI, _PD]
        l.sfeec_ref_transpose.argtypes = [C.c_int, C.c_int, _PI, _PI, _PD, _PI, _PI, _PD]
        l.sfeec_ref_cubical_curl.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double,
                                             C.c_double, C.c_double, _PI, _PI, _PD]
        l.sfeec_ref_yee_create.restype = C.c_void_p
        l.sfeec_ref_yee_create.argtypes = [C.c_int] * 3 + [C.c_double] * 3
        l.sfeec_ref_yee_destroy.argtypes = [C.c_void_p]
        l.sfeec_ref_yee_set.argtypes = [C.c_void_p, C.c_int, _PD]
        l.sfeec_ref_yee_get.argtypes = [C.c_void_p, C.c_int, _PD]
        l.sfeec_ref_yee_step.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double,
                                         C.c_int]
        l.sfeec_ref_yee_advance_b.argtypes = [C.c_void_p, C.c_double]
        _ref = l
    return _ref


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _ip(a):
    return a.ctypes.data_as(_PI)


def ref_cubical_curl(nx, ny, nz, dx, dy, dz):
    """Q1 curl of the reference periodic lattice (mesh_cubical.cpp + operators.cpp:37)."""
    l = ref_lib()
    nnz = l.sfeec_ref_cubical_curl(nx, ny, nz, dx, dy, dz, None, None, None)
    n = 3 * nx * ny * nz
    rp, ci, va = np.zeros(n + 1, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz)
    l.sfeec_ref_cubical_curl(nx, ny, nz, dx, dy, dz, _ip(rp), _ip(ci), _d(va))
    return (n, n, rp.astype(np.int64), ci, va)


def ref_from_triplets(rows, cols, r, c, v):
    l = ref_lib()
    r, c, v = _i32(r), _i32(c), np.ascontiguousarray(v, np.float64)
    nnz = l.sfeec_ref_from_triplets(rows, cols, r.size, _ip(r), _ip(c), _d(v), None, None, None)
    if nnz < 0:
        raise ValueError(l.sfeec_ref_last_error().decode())
    rp, ci, va = np.zeros(rows + 1, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz)
    l.sfeec_ref_from_triplets(rows, cols, r.size, _ip(r), _ip(c), v.ctypes.data_as(_PD),
                              _ip(rp), _ip(ci), va.ctypes.data_as(_PD))
    return (rows, cols, rp.astype(np.int64), ci, va)


def ref_transpose(a):
    rows, cols, rp, ci, va = a
    l = ref_lib()
    trp, tci, tva = np.zeros(cols + 1, np.int32), np.zeros(ci.size, np.int32), np.zeros(ci.size)
    rp32, ci32 = _i32(rp), _i32(ci)
    va = np.ascontiguousarray(va, np.float64)
    l.sfeec_ref_transpose(rows, cols, _ip(rp32), _ip(ci32), va.ctypes.data_as(_PD), _ip(trp),
                          _ip(tci), tva.ctypes.data_as(_PD))
    return (cols, rows, trp.astype(np.int64), tci, tva)


def ref_spmv(a, x):
    rows, cols, rp, ci, va = a
    y = np.zeros(rows)
    rp32, ci32 = _i32(rp), _i32(ci)
    va = np.ascontiguousarray(va, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    ref_lib().sfeec_ref_spmv(rows, cols, _ip(rp32), _ip(ci32), va.ctypes.data_as(_PD),
                             x.ctypes.data_as(_PD), y.ctypes.data_as(_PD))
    return y


# --------------------------------------------------------------------------
# the reference's setup code (make_pattern, SPAI, Q1 operators)
# --------------------------------------------------------------------------
REFSETUP_PATH = os.path.join(HERE, "_ref", "libsfeec_ref_setup.so")
_refs = None


def refsetup_available() -> bool:
    return os.path.exists(REFSETUP_PATH)


def refs_lib():
    global _refs
    if _refs is None:
        l = C.CDLL(REFSETUP_PATH)
        l.sfeec_refs_last_error.restype = C.c_char_p
        for f in ("sfeec_refs_pattern", "sfeec_refs_spai", "sfeec_refs_cubical"):
            getattr(l, f).restype = C.c_void_p
        l.sfeec_refs_pattern.argtypes = [C.c_int, _PI, _PI, _PD, C.c_int]
        l.sfeec_refs_spai.argtypes = [C.c_int, _PI, _PI, _PD, C.c_int, C.c_int]
        l.sfeec_refs_cubical.argtypes = [C.c_int] * 3 + [C.c_double] * 3 + [C.c_int]
        for f in ("sfeec_refs_op_rows", "sfeec_refs_op_cols", "sfeec_refs_op_nnz",
                  "sfeec_refs_op_destroy"):
            getattr(l, f).argtypes = [C.c_void_p]
        l.sfeec_refs_op_export.argtypes = [C.c_void_p, _PI, _PI, _PD, _PD]
        _refs = l
    return _refs


def _refs_take(h):
    """(rows, cols, row_ptr, col_idx, val), report from an operator handle."""
    l = refs_lib()
    if not h:
        raise ValueError(l.sfeec_refs_last_error().decode())
    rows, cols, nnz = l.sfeec_refs_op_rows(h), l.sfeec_refs_op_cols(h), l.sfeec_refs_op_nnz(h)
    rp, ci, va = np.zeros(rows + 1, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz)
    rep = np.zeros(4)
    l.sfeec_refs_op_export(h, _ip(rp), _ip(ci), va.ctypes.data_as(_PD), rep.ctypes.data_as(_PD))
    l.sfeec_refs_op_destroy(h)
    return (rows, cols, rp.astype(np.int64), ci, va), rep


_PATTERN_KINDS = {"diagonal": 0, "m1": 1, "m1sq": 2, "dense": 3}


def ref_make_pattern(m, kind):
    """The reference's make_pattern (spai.cpp:31-72) of a symmetric operator
    m = (rows, cols, row_ptr, col_idx, val): row l = the index set I_l."""
    rows, _, rp, ci, va = m
    va = np.ascontiguousarray(va, np.float64)
    h = refs_lib().sfeec_refs_pattern(rows, _ip(_i32(rp)), _ip(_i32(ci)), va.ctypes.data_as(_PD),
                                      _PATTERN_KINDS[kind])
    return _refs_take(h)[0]


def ref_spai(m, kind, use_cg=False):
    """The reference's spai_approximate_inverse (spai.cpp:127-286) on
    make_pattern(m, kind) -> (Q, report dict)."""
    rows, _, rp, ci, va = m
    va = np.ascontiguousarray(va, np.float64)
    h = refs_lib().sfeec_refs_spai(rows, _ip(_i32(rp)), _ip(_i32(ci)), va.ctypes.data_as(_PD),
                                   _PATTERN_KINDS[kind], 1 if use_cg else 0)
    q, rep = _refs_take(h)
    return q, {"frobenius_residual": rep[0], "avg_nnz_per_row": rep[1],
               "max_column_residual": rep[2], "fallback_columns": int(rep[3])}


def ref_cubical_operator(nx, ny, nz, dx, dy, dz, which):
    """Q1 operators of the reference's periodic lattice from its own
    build_space + derivative_matrix / mass_matrix: 'c', 'm1', 'm2' or 'd'."""
    k = {"c": 0, "m1": 1, "m2": 2, "d": 3}[which]
    return _refs_take(refs_lib().sfeec_refs_cubical(nx, ny, nz, dx, dy, dz, k))[0]


class RefScheme:
    """The reference SplitScheme (dynamics.cpp) on CSR tuples (rows, cols, rp, ci, val)."""

    def __init__(self, strang, dt, q, c, m2, eps0=1.0, mu0=1.0, div=None, warn_cfl=False):
        l = ref_lib()
        self._keep = []

        def arrs(a):
            rp, ci = _i32(a[2]), _i32(a[3])
            va = np.ascontiguousarray(a[4], np.float64)
            self._keep += [rp, ci, va]
            return _ip(rp), _ip(ci), va.ctypes.data_as(_PD)

        qa, ca, ma = arrs(q), arrs(c), arrs(m2)
        da = arrs(div) if div is not None else (None, None, None)
        self.h = l.sfeec_ref_scheme_create(
            1 if strang else 0, dt, q[0], *qa, c[0], c[1], *ca, *ma, eps0, mu0,
            div[0] if div is not None else 0, *da, 1 if warn_cfl else 0)
        if not self.h:
            raise ValueError(l.sfeec_ref_last_error().decode())
        self.n1, self.n2 = c[1], c[0]
        self.keep_ops = (q, c, m2, div)

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().sfeec_ref_scheme_destroy(self.h)
            self.h = None

    def q_sym(self):
        l = ref_lib()
        nnz = l.sfeec_ref_scheme_qsym_nnz(self.h)
        rp, ci, va = np.zeros(self.n1 + 1, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz)
        l.sfeec_ref_scheme_qsym(self.h, _ip(rp), _ip(ci), va.ctypes.data_as(_PD))
        return (self.n1, self.n1, rp.astype(np.int64), ci, va)

    def steps(self, be, first, e, nsteps, time=0.0, energy=False):
        first = np.array(first, dtype=np.float64)
        e = np.array(e, dtype=np.float64)
        t = C.c_double(time)
        hist = np.zeros(max(nsteps, 1)) if energy else None
        secs = C.c_double()
        code = ref_lib().sfeec_ref_scheme_steps(
            self.h, 1 if be else 0, first.ctypes.data_as(_PD), first.size,
            e.ctypes.data_as(_PD), e.size, C.byref(t), nsteps,
            hist.ctypes.data_as(_PD) if energy else None, C.byref(secs))
        if code:
            raise ValueError(ref_lib().sfeec_ref_last_error().decode())
        self.last_seconds = secs.value
        return first, e, t.value, (hist[:nsteps] if energy else None)

    def flow(self, which, be, first, e, dt):
        first = np.array(first, dtype=np.float64)
        e = np.array(e, dtype=np.float64)
        code = ref_lib().sfeec_ref_scheme_flow(self.h, which, 1 if be else 0,
                                               first.ctypes.data_as(_PD), first.size,
                                               e.ctypes.data_as(_PD), e.size, dt)
        if code:
            raise ValueError(ref_lib().sfeec_ref_last_error().decode())
        return first, e

    def energy(self, be, first, e):
        out = C.c_double()
        first = np.ascontiguousarray(first, np.float64)
        e = np.ascontiguousarray(e, np.float64)
        ref_lib().sfeec_ref_scheme_energy(self.h, 1 if be else 0, first.ctypes.data_as(_PD),
                                          first.size, e.ctypes.data_as(_PD), e.size,
                                          C.byref(out))
        return out.value

    def gauss(self, first, e):
        out = C.c_double()
        first = np.ascontiguousarray(first, np.float64)
        e = np.ascontiguousarray(e, np.float64)
        code = ref_lib().sfeec_ref_scheme_gauss(self.h, 1, first.ctypes.data_as(_PD),
                                                first.size, e.ctypes.data_as(_PD), e.size,
                                                C.byref(out))
        if code:
            raise ValueError(ref_lib().sfeec_ref_last_error().decode())
        return out.value

    def cfl(self):
        out = C.c_double()
        ref_lib().sfeec_ref_scheme_cfl(self.h, C.byref(out))
        return out.value


class RefYee:
    """YeeGrid + yee_fdtd_step (yee.cpp:9-74)."""

    def __init__(self, nx, ny, nz, dx, dy, dz):
        self.h = ref_lib().sfeec_ref_yee_create(nx, ny, nz, dx, dy, dz)
        self.n = 3 * nx * ny * nz

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().sfeec_ref_yee_destroy(self.h)
            self.h = None

    def set(self, e, b):
        ref_lib().sfeec_ref_yee_set(self.h, 0, _d(e))
        ref_lib().sfeec_ref_yee_set(self.h, 1, _d(b))

    def get(self):
        e, b = np.zeros(self.n), np.zeros(self.n)
        ref_lib().sfeec_ref_yee_get(self.h, 0, e.ctypes.data_as(_PD))
        ref_lib().sfeec_ref_yee_get(self.h, 1, b.ctypes.data_as(_PD))
        return e, b

    def step(self, dt, n=1, eps0=1.0, mu0=1.0):
        ref_lib().sfeec_ref_yee_step(self.h, dt, eps0, mu0, n)

    def advance_b(self, dt):
        ref_lib().sfeec_ref_yee_advance_b(self.h, dt)


# --------------------------------------------------------------------------
# plain-C restatement
# --------------------------------------------------------------------------
class or_csr(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("row_ptr", _PI64),
                ("col_idx", _PI32), ("val", _PD)]


class or_scheme(C.Structure):
    _fields_ = [("strang", C.c_int), ("be", C.c_int), ("dt", C.c_double),
                ("eps0", C.c_double), ("mu0", C.c_double), ("q_sym", or_csr), ("c", or_csr),
                ("ct", or_csr), ("m2", or_csr), ("div", C.POINTER(or_csr))]


_port = None


def port_lib():
    global _port
    if _port is None:
        l = C.CDLL(PORT_PATH)
        l.or_spmv.argtypes = [C.POINTER(or_csr), _PD, _PD]
        l.or_from_triplets.restype = C.c_int64
        l.or_from_triplets.argtypes = [C.c_int64, C.c_int64, _PI32, _PI32, _PD, _PI64, _PI32,
                                       _PD]
        l.or_symmetric_part.restype = C.c_int64
        l.or_symmetric_part.argtypes = [C.POINTER(or_csr), _PI64, _PI32, _PD]
        l.or_transpose.argtypes = [C.POINTER(or_csr), _PI64, _PI32, _PD]
        for f in ("or_flow_he", "or_flow_ha"):
            getattr(l, f).argtypes = [C.POINTER(or_scheme), _PD, _PD, C.c_double]
        l.or_steps.argtypes = [C.POINTER(or_scheme), _PD, _PD, C.c_int64, _PD]
        l.or_energy.restype = C.c_double
        l.or_energy.argtypes = [C.POINTER(or_scheme), _PD, _PD]
        l.or_gauss_residual.restype = C.c_double
        l.or_gauss_residual.argtypes = [C.POINTER(or_scheme), _PD]
        l.or_cfl_number.restype = C.c_double
        l.or_cfl_number.argtypes = [C.POINTER(or_scheme)]
        l.or_rng_fill_uniform.argtypes = [C.c_uint64, C.c_double, C.c_double, _PD, C.c_int64]
        l.or_yee_advance_e.argtypes = [C.c_int] * 3 + [_PD, _PD, _PD, C.c_double, C.c_double]
        l.or_yee_advance_b.argtypes = [C.c_int] * 3 + [_PD, _PD, _PD, C.c_double]
        l.to_build.restype = C.c_int
        l.to_build.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int] + \
            [C.POINTER(to_csr)] * 5 + [_PI64]
        l.to_free.argtypes = [C.POINTER(to_csr)]
        _port = l
    return _port


class to_csr(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64),
                ("rp", _PI64), ("ci", _PI32), ("v", _PD)]


TET_OPERATORS = ("c", "d", "m1", "m2", "q_sym")


def tet_c_operators(n, jitter, seed, want=("c", "m2", "q_sym")):
    """The 3-D Kuhn tet operators from the C restatement (oracle/tet_oracle.c):
    dict name -> (rows, cols, row_ptr, col_idx, val), plus "counts" =
    (N1, N2, T, SPAI columns that failed the pivot test). Test / reference-arm
    infrastructure only."""
    l = port_lib()
    mask = sum(1 << TET_OPERATORS.index(w) for w in want)
    outs = [to_csr() for _ in TET_OPERATORS]
    counts = np.zeros(4, np.int64)
    rc = l.to_build(int(n), float(jitter), int(seed), mask, *[C.byref(o) for o in outs],
                    counts.ctypes.data_as(_PI64))
    res = {"counts": tuple(int(x) for x in counts)}
    try:
        if rc != 0:
            raise MemoryError("tet_oracle: allocation failed or bad arguments")
        for name, o in zip(TET_OPERATORS, outs):
            if name not in want:
                continue
            rp = np.ctypeslib.as_array(o.rp, (o.rows + 1,)).copy()
            ci = np.ctypeslib.as_array(o.ci, (max(o.nnz, 1),))[:o.nnz].copy()
            va = np.ctypeslib.as_array(o.v, (max(o.nnz, 1),))[:o.nnz].copy()
            res[name] = (int(o.rows), int(o.cols), rp, ci, va)
    finally:
        for o in outs:
            l.to_free(C.byref(o))
    return res


class _Csr:
    """Keeps numpy buffers alive behind an or_csr view."""

    def __init__(self, a):
        rows, cols, rp, ci, va = a
        self.rp = np.ascontiguousarray(rp, np.int64)
        self.ci = np.ascontiguousarray(ci, np.int32)
        self.va = np.ascontiguousarray(va, np.float64)
        self.s = or_csr(rows, cols, self.rp.ctypes.data_as(_PI64), self.ci.ctypes.data_as(_PI32),
                        self.va.ctypes.data_as(_PD))


def port_uniform(seed, n, lo=-1.0, hi=1.0):
    """Rng(seed).uniform(lo, hi) x n (core.hpp:44-63)."""
    out = np.zeros(n)
    port_lib().or_rng_fill_uniform(seed, lo, hi, out.ctypes.data_as(_PD), n)
    return out


def port_spmv(a, x):
    m = _Csr(a)
    y = np.zeros(a[0])
    x = np.ascontiguousarray(x, np.float64)
    port_lib().or_spmv(C.byref(m.s), x.ctypes.data_as(_PD), y.ctypes.data_as(_PD))
    return y


def port_from_triplets(rows, cols, r, c, v):
    l = port_lib()
    r = np.ascontiguousarray(r, np.int32)
    c = np.ascontiguousarray(c, np.int32)
    v = np.ascontiguousarray(v, np.float64)
    args = (r.ctypes.data_as(_PI32), c.ctypes.data_as(_PI32), v.ctypes.data_as(_PD))
    nnz = l.or_from_triplets(rows, r.size, *args, None, None, None)
    rp, ci, va = np.zeros(rows + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz)
    l.or_from_triplets(rows, r.size, *args, rp.ctypes.data_as(_PI64), ci.ctypes.data_as(_PI32),
                       va.ctypes.data_as(_PD))
    return (rows, cols, rp, ci, va)


def port_symmetric_part(q):
    m = _Csr(q)
    l = port_lib()
    nnz = l.or_symmetric_part(C.byref(m.s), None, None, None)
    rp, ci, va = np.zeros(q[0] + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz)
    l.or_symmetric_part(C.byref(m.s), rp.ctypes.data_as(_PI64), ci.ctypes.data_as(_PI32),
                        va.ctypes.data_as(_PD))
    return (q[0], q[1], rp, ci, va)


def port_transpose(a):
    m = _Csr(a)
    rp, ci, va = np.zeros(a[1] + 1, np.int64), np.zeros(a[3].size, np.int32), np.zeros(a[3].size)
    port_lib().or_transpose(C.byref(m.s), rp.ctypes.data_as(_PI64), ci.ctypes.data_as(_PI32),
                            va.ctypes.data_as(_PD))
    return (a[1], a[0], rp, ci, va)


class PortScheme:
    """The C restatement of SplitScheme. q is symmetrised like the reference ctor."""

    def __init__(self, strang, dt, q, c, m2, eps0=1.0, mu0=1.0, div=None, be=True,
                 q_is_symmetric=False):
        qs = q if q_is_symmetric else port_symmetric_part(q)
        self.ops = [_Csr(qs), _Csr(c), _Csr(port_transpose(c)), _Csr(m2)]
        self.div = _Csr(div) if div is not None else None
        self.s = or_scheme(1 if strang else 0, 1 if be else 0, dt, eps0, mu0,
                           self.ops[0].s, self.ops[1].s, self.ops[2].s, self.ops[3].s,
                           C.pointer(self.div.s) if self.div else None)
        self.q_sym = qs

    def steps(self, first, e, nsteps, energy=False):
        first = np.array(first, dtype=np.float64)
        e = np.array(e, dtype=np.float64)
        hist = np.zeros(max(nsteps, 1)) if energy else None
        port_lib().or_steps(C.byref(self.s), first.ctypes.data_as(_PD), e.ctypes.data_as(_PD),
                            nsteps, hist.ctypes.data_as(_PD) if energy else None)
        return first, e, (hist[:nsteps] if energy else None)

    def flow_he(self, first, e, dt):
        first, e = np.array(first, np.float64), np.array(e, np.float64)
        port_lib().or_flow_he(C.byref(self.s), first.ctypes.data_as(_PD),
                              e.ctypes.data_as(_PD), dt)
        return first, e

    def flow_ha(self, first, e, dt):
        first, e = np.array(first, np.float64), np.array(e, np.float64)
        port_lib().or_flow_ha(C.byref(self.s), first.ctypes.data_as(_PD),
                              e.ctypes.data_as(_PD), dt)
        return first, e

    def energy(self, first, e):
        first, e = np.ascontiguousarray(first, np.float64), np.ascontiguousarray(e, np.float64)
        return port_lib().or_energy(C.byref(self.s), first.ctypes.data_as(_PD),
                                    e.ctypes.data_as(_PD))

    def gauss(self, b):
        b = np.ascontiguousarray(b, np.float64)
        return port_lib().or_gauss_residual(C.byref(self.s), b.ctypes.data_as(_PD))

    def cfl(self):
        return port_lib().or_cfl_number(C.byref(self.s))


def port_yee_step(nx, ny, nz, d, e, b, dt, nsteps=1, c2=1.0):
    """yee_fdtd_step x nsteps (yee.cpp:71-74) on component-major arrays."""
    e = np.array(e, np.float64)
    b = np.array(b, np.float64)
    dd = np.ascontiguousarray(d, np.float64)
    l = port_lib()
    for _ in range(nsteps):
        l.or_yee_advance_e(nx, ny, nz, dd.ctypes.data_as(_PD), e.ctypes.data_as(_PD),
                           b.ctypes.data_as(_PD), dt, c2)
        l.or_yee_advance_b(nx, ny, nz, dd.ctypes.data_as(_PD), e.ctypes.data_as(_PD),
                           b.ctypes.data_as(_PD), dt)
    return e, b


def port_yee_advance_b(nx, ny, nz, d, e, b, dt):
    b = np.array(b, np.float64)
    dd = np.ascontiguousarray(d, np.float64)
    e = np.ascontiguousarray(e, np.float64)
    port_lib().or_yee_advance_b(nx, ny, nz, dd.ctypes.data_as(_PD), e.ctypes.data_as(_PD),
                                b.ctypes.data_as(_PD), dt)
    return b
