"""Host-side mirror of the reference's operator/step interface.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/sfeec/{sparse,dynamics,yee}.hpp so the parity
tests read like the reference's own tests:

  SparseOperator          sparse.hpp:14-33 (CSR, sorted columns, no zeros)
  operator_from_triplets  sparse.cpp:20-61
  scaled_identity         sparse.cpp:63-73
  transpose               sparse.cpp:75-94
  UnitSystem, FieldState, make_state    dynamics.hpp:9-25, dynamics.cpp:135-143
  SplitScheme             dynamics.hpp:31-67 -- every compute call runs on the
                          B200 through the C ABI (include/sfeec_b200.h)
  YeeScheme               the lumped-mass (Yee) special case, yee.hpp:12-37

The step itself never runs on the CPU here: there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._lib import InvalidParameter, DeviceError  # noqa: F401  (re-export)


class Formulation(enum.IntEnum):
    AE = L.FORM_AE
    BE = L.FORM_BE


class SplitKind(enum.IntEnum):
    LieTrotter = L.SPLIT_LIE_TROTTER
    Strang = L.SPLIT_STRANG


@dataclass
class UnitSystem:
    eps0: float = 1.0
    mu0: float = 1.0

    def c2(self) -> float:
        return 1.0 / (self.eps0 * self.mu0)


@dataclass
class SparseOperator:
    """CSR operator, int64 row pointers, int32 columns, fp64 values."""

    rows: int
    cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    val: np.ndarray
    symmetric: bool = False

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int32)
        self.val = np.ascontiguousarray(self.val, dtype=np.float64)

    def nnz(self) -> int:
        return int(self.col_idx.size)

    def row_cols(self, r: int) -> np.ndarray:
        return self.col_idx[self.row_ptr[r]:self.row_ptr[r + 1]]

    def row_vals(self, r: int) -> np.ndarray:
        return self.val[self.row_ptr[r]:self.row_ptr[r + 1]]

    def at(self, r: int, c: int) -> float:
        cs = self.row_cols(r)
        k = np.searchsorted(cs, c)
        if k < cs.size and cs[k] == c:
            return float(self.row_vals(r)[k])
        return 0.0

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols))
        rows = np.repeat(np.arange(self.rows), np.diff(self.row_ptr))
        d[rows, self.col_idx] = self.val
        return d

    def view(self) -> L.sfeec_csr:
        v = L.sfeec_csr()
        v.rows, v.cols = self.rows, self.cols
        v.row_ptr = L.i64ptr(self.row_ptr)
        v.col_idx = L.i32ptr(self.col_idx)
        v.val = L.dptr(self.val)
        return v

    @staticmethod
    def _from_owned(m: L.sfeec_csr_owned, symmetric=False) -> "SparseOperator":
        rows, cols, rp, ci, va = L.owned_to_numpy(m)
        return SparseOperator(rows, cols, rp, ci, va, symmetric)


def operator_from_triplets(rows, cols, r, c, v, symmetric=False) -> SparseOperator:
    """sparse.cpp:20-61 (deterministic, duplicates summed in input order)."""
    r = np.ascontiguousarray(r, dtype=np.int32)
    c = np.ascontiguousarray(c, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = L.sfeec_csr_owned()
    L.check(L.lib().sfeec_csr_from_triplets(rows, cols, r.size, L.i32ptr(r), L.i32ptr(c),
                                            L.dptr(v), C.byref(out)))
    return SparseOperator._from_owned(out, symmetric)


def scaled_identity(n: int, s: float) -> SparseOperator:
    """sparse.cpp:63-73."""
    return SparseOperator(n, n, np.arange(n + 1), np.arange(n), np.full(n, float(s)), True)


def transpose(a: SparseOperator) -> SparseOperator:
    out = L.sfeec_csr_owned()
    v = a.view()
    L.check(L.lib().sfeec_csr_transpose(C.byref(v), C.byref(out)))
    return SparseOperator._from_owned(out, a.symmetric)


def symmetric_part(q: SparseOperator) -> SparseOperator:
    """dynamics.cpp:10-25."""
    out = L.sfeec_csr_owned()
    v = q.view()
    L.check(L.lib().sfeec_csr_symmetric_part(C.byref(v), C.byref(out)))
    return SparseOperator._from_owned(out, True)


@dataclass
class FieldState:
    formulation: Formulation = Formulation.AE
    first: np.ndarray = field(default_factory=lambda: np.zeros(0))
    e: np.ndarray = field(default_factory=lambda: np.zeros(0))
    time: float = 0.0

    def copy(self) -> "FieldState":
        return FieldState(self.formulation, self.first.copy(), self.e.copy(), self.time)


def make_state(f: Formulation, first, e, time: float = 0.0) -> FieldState:
    return FieldState(Formulation(f), np.array(first, dtype=np.float64),
                      np.array(e, dtype=np.float64), float(time))


class SplitScheme:
    """dynamics.hpp:31-67 on a B200: operators and state live in HBM.

    The formulation is fixed at construction (the device keeps one resident
    state layout); states of the other formulation raise InvalidParameter.
    `strict=True` selects the bitwise-reference kernels (SFEEC_STRICT).
    """

    def __init__(self, kind: SplitKind, dt: float, q: SparseOperator, c: SparseOperator,
                 m2: SparseOperator, units: UnitSystem | None = None,
                 div: SparseOperator | None = None, warn_cfl: bool = True, *,
                 formulation: Formulation = Formulation.BE, strict: bool = False,
                 q_is_symmetric: bool = False, device: int = 0):
        units = units or UnitSystem()
        self._kind, self._dt, self._units = SplitKind(kind), float(dt), units
        self._formulation = Formulation(formulation)
        self._c, self._m2 = c, m2
        flags = (L.STRICT if strict else 0) | (0 if warn_cfl else L.NO_CFL_WARN)
        flags |= L.Q_IS_SYMMETRIC if q_is_symmetric else 0
        h = C.c_void_p()
        qv, cv, mv = q.view(), c.view(), m2.view()
        dv = div.view() if div is not None else None
        L.check(L.lib().sfeec_dev_create(
            C.byref(qv), C.byref(cv), C.byref(mv), C.byref(dv) if dv is not None else None,
            self._dt, units.eps0, units.mu0, int(self._kind), int(self._formulation), device,
            flags, C.byref(h)))
        self._h = h
        self._n1, self._n2 = c.cols, c.rows

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and callable(getattr(L, "lib", None)):  # (module globals go at shutdown)
            L.lib().sfeec_dev_destroy(h)
            self._h = None

    # accessors (dynamics.hpp:38-45)
    def kind(self):
        return self._kind

    def dt(self):
        return self._dt

    def units(self):
        return self._units

    def q_sym(self) -> SparseOperator:
        nnz = C.c_int64()
        L.check(L.lib().sfeec_dev_q_sym(self._h, C.byref(nnz), None, None, None))
        rp = np.zeros(self._n1 + 1, np.int64)
        ci = np.zeros(nnz.value, np.int32)
        va = np.zeros(nnz.value)
        L.check(L.lib().sfeec_dev_q_sym(self._h, None, L.i64ptr(rp), L.i32ptr(ci), L.dptr(va)))
        return SparseOperator(self._n1, self._n1, rp, ci, va, True)

    def curl(self):
        return self._c

    def m2(self):
        return self._m2

    # state transfer
    def _check_state(self, s: FieldState):
        if s.formulation != self._formulation:
            raise InvalidParameter("SplitScheme: state formulation differs from the device's")
        nf = self._n2 if self._formulation == Formulation.BE else self._n1
        if s.first.size != nf or s.e.size != self._n1:
            raise InvalidParameter("spmv: dimension mismatch")

    def load(self, s: FieldState) -> None:
        self._check_state(s)
        first = np.ascontiguousarray(s.first, dtype=np.float64)
        e = np.ascontiguousarray(s.e, dtype=np.float64)
        L.check(L.lib().sfeec_dev_set_state(self._h, L.dptr(first), first.size, L.dptr(e),
                                            e.size, s.time))

    def fetch(self) -> FieldState:
        nf = self._n2 if self._formulation == Formulation.BE else self._n1
        first, e, t = np.zeros(nf), np.zeros(self._n1), C.c_double()
        L.check(L.lib().sfeec_dev_get_state(self._h, L.dptr(first), L.dptr(e), C.byref(t)))
        return FieldState(self._formulation, first, e, t.value)

    # exact sub-flows, dynamics.cpp:47-67 (in place, clock untouched)
    def flow_he(self, s: FieldState, dt: float) -> None:
        self.load(s)
        L.check(L.lib().sfeec_dev_flow_he(self._h, float(dt)))
        out = self.fetch()
        s.first[:], s.e[:] = out.first, out.e

    def flow_ha(self, s: FieldState, dt: float) -> None:
        self.load(s)
        L.check(L.lib().sfeec_dev_flow_ha(self._h, float(dt)))
        out = self.fetch()
        s.first[:], s.e[:] = out.first, out.e

    def step(self, s: FieldState) -> FieldState:
        """dynamics.cpp:69-90: returns a new state one step later."""
        return self.advance(s, 1)

    def advance(self, s: FieldState, nsteps: int) -> FieldState:
        """nsteps x step with the state resident on the device."""
        self.load(s)
        L.check(L.lib().sfeec_dev_advance(self._h, int(nsteps)))
        return self.fetch()

    # resident-state forms: no host round trip of the state
    def advance_resident(self, nsteps: int) -> None:
        L.check(L.lib().sfeec_dev_advance(self._h, int(nsteps)))

    def energy_resident(self) -> float:
        out = C.c_double()
        L.check(L.lib().sfeec_dev_energy(self._h, C.byref(out)))
        return out.value

    def flow_he_resident(self, dt: float) -> None:
        L.check(L.lib().sfeec_dev_flow_he(self._h, float(dt)))

    def flow_ha_resident(self, dt: float) -> None:
        L.check(L.lib().sfeec_dev_flow_ha(self._h, float(dt)))

    def advance_diag(self, s: FieldState, nsteps: int, diag_every: int = 1):
        """advance + energy and Gauss residual after every diag_every steps."""
        self.load(s)
        n = nsteps // diag_every
        en, ga = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        L.check(L.lib().sfeec_dev_advance_diag(self._h, int(nsteps), int(diag_every),
                                               L.dptr(en), L.dptr(ga)))
        return self.fetch(), en[:n], ga[:n]

    def energy(self, s: FieldState) -> float:
        self.load(s)
        out = C.c_double()
        L.check(L.lib().sfeec_dev_energy(self._h, C.byref(out)))
        return out.value

    def gauss_residual(self, s: FieldState) -> float:
        if s.formulation != Formulation.BE:
            raise InvalidParameter("gauss_residual: (b, e) formulation required")
        self.load(s)
        out = C.c_double()
        L.check(L.lib().sfeec_dev_gauss_residual(self._h, C.byref(out)))
        return out.value

    def cfl_number(self) -> float:
        out = C.c_double()
        L.check(L.lib().sfeec_dev_cfl_number(self._h, C.byref(out)))
        return out.value

    # device-resident handles for benchmarks
    @property
    def handle(self):
        return self._h

    def step_bytes(self) -> float:
        return L.lib().sfeec_dev_step_bytes(self._h)

    def curl_of_curl(self, a: np.ndarray) -> np.ndarray:
        """apply_curl_of_curl (operators.cpp:268-290): Q_sym C^T M2 C a on the device."""
        a = np.ascontiguousarray(a, np.float64)
        if a.size != self._n1:
            raise InvalidParameter("apply_curl_of_curl: dimension mismatch")
        y = np.zeros(self._n1)
        L.check(L.lib().sfeec_dev_curl_curl(self._h, L.dptr(a), L.dptr(y)))
        return y

    def apply(self, which: str, x: np.ndarray) -> np.ndarray:
        """y = A x with a resident operator: 'q_sym', 'c', 'ct', 'm2' or 'div'."""
        idx = {"q_sym": 0, "c": 1, "ct": 2, "m2": 3, "div": 4}[which]
        rows = {"q_sym": self._n1, "c": self._n2, "ct": self._n1, "m2": self._n2}
        x = np.ascontiguousarray(x, np.float64)
        n_out = rows.get(which)
        if n_out is None:  # div: cells; ask via a probe-free bound
            n_out = getattr(self, "n_tets", None)
            if n_out is None:
                raise InvalidParameter("apply('div') needs the cell count")
        y = np.zeros(n_out)
        L.check(L.lib().sfeec_dev_apply(self._h, idx, L.dptr(x), L.dptr(y)))
        return y

    def layout_info(self, which: str) -> dict:
        """Device layout of a resident operator (sfeec_dev_layout_info)."""
        idx = {"q_sym": 0, "c": 1, "ct": 2, "m2": 3, "div": 4}[which]
        info, by = np.zeros(9, np.int64), C.c_double()
        L.check(L.lib().sfeec_dev_layout_info(self._h, idx, L.i64ptr(info), C.byref(by)))
        keys = ("layout", "delta", "ell", "slices", "full_slices", "entries", "nnz", "win",
                "units")
        out = {k: int(v) for k, v in zip(keys, info)}
        out["stream_bytes"] = by.value
        return out

    def set_dt(self, dt: float) -> None:
        L.check(L.lib().sfeec_dev_set_dt(self._h, float(dt)))
        self._dt = float(dt)

    def last_launches(self) -> int:
        return int(L.lib().sfeec_dev_last_launches(self._h))

    KERNEL_CLASSES = ("K-Q", "K-Cb", "K-CTe", "K-M2", "other")

    def kernel_timing(self, enable: bool = True) -> dict:
        """Per-kernel device time since the last call (then (dis)arm timing)."""
        ms, n, by = np.zeros(5), np.zeros(5, np.int64), np.zeros(5)
        L.check(L.lib().sfeec_dev_kernel_timing(self._h, 1 if enable else 0, L.dptr(ms),
                                                L.i64ptr(n), L.dptr(by)))
        return {k: {"ms": ms[i], "launches": int(n[i]), "bytes_per_launch": by[i]}
                for i, k in enumerate(self.KERNEL_CLASSES)}


class YeeScheme:
    """Lumped-mass SFEEC on an nx x ny x nz lattice (Q = I/dV, M2 = dV I).

    State is the (b, e) pair in the sfeec_yee numbering (yee_layout.hpp):
    periodic = the reference's axis-major ids; PEC = interior edges + all
    faces. precision 8 or 4 (fp64 / fp32 fields on the device).
    """

    def __init__(self, nx, ny, nz, dx, dy, dz, dt, units: UnitSystem | None = None,
                 bc: int = L.BC_PEC, precision: int = 8, device: int = 0):
        units = units or UnitSystem()
        h = C.c_void_p()
        L.check(L.lib().sfeec_yee_create(nx, ny, nz, dx, dy, dz, dt, units.eps0, units.mu0, bc,
                                         precision, device, C.byref(h)))
        self._h = h
        ne, nf = C.c_int64(), C.c_int64()
        L.check(L.lib().sfeec_yee_dof_counts(h, C.byref(ne), C.byref(nf)))
        self.n_edges, self.n_faces = ne.value, nf.value
        self.dt = dt

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and callable(getattr(L, "lib", None)):  # (module globals go at shutdown)
            L.lib().sfeec_yee_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def set_variant(self, v: int) -> None:
        L.check(L.lib().sfeec_yee_set_variant(self._h, v))

    def load(self, b, e, time=0.0):
        b = np.ascontiguousarray(b, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
        if b.size != self.n_faces or e.size != self.n_edges:
            raise InvalidParameter("spmv: dimension mismatch")
        L.check(L.lib().sfeec_yee_set_state(self._h, L.dptr(b), L.dptr(e), float(time)))

    def fetch(self):
        b, e, t = np.zeros(self.n_faces), np.zeros(self.n_edges), C.c_double()
        L.check(L.lib().sfeec_yee_get_state(self._h, L.dptr(b), L.dptr(e), C.byref(t)))
        return b, e, t.value

    def advance(self, nsteps: int) -> None:
        L.check(L.lib().sfeec_yee_advance(self._h, int(nsteps)))

    def flow_he(self, dt: float) -> None:
        L.check(L.lib().sfeec_yee_flow_he(self._h, float(dt)))

    def flow_ha(self, dt: float) -> None:
        L.check(L.lib().sfeec_yee_flow_ha(self._h, float(dt)))

    def energy(self) -> float:
        out = C.c_double()
        L.check(L.lib().sfeec_yee_energy(self._h, C.byref(out)))
        return out.value

    def step_bytes(self) -> float:
        return L.lib().sfeec_yee_step_bytes(self._h)

    def last_launches(self) -> int:
        return int(L.lib().sfeec_yee_last_launches(self._h))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    L.check(L.lib().sfeec_nccl_unique_id(buf))
    return buf.raw


def yee_slab_dofs(nx, ny, nz, rank, nranks):
    """(edge_map, face_map): local DOF -> global DOF of z-slab `rank`."""
    ne, nf = C.c_int64(), C.c_int64()
    L.check(L.lib().sfeec_yee_slab_dof_counts(nx, ny, nz, rank, nranks, C.byref(ne),
                                              C.byref(nf)))
    em, fm = np.zeros(ne.value, np.int64), np.zeros(nf.value, np.int64)
    L.check(L.lib().sfeec_yee_slab_dof_map(nx, ny, nz, rank, nranks, L.i64ptr(em),
                                           L.i64ptr(fm)))
    return em, fm


class YeeSlab(YeeScheme):
    """One z-slab of a PEC Yee lattice per process; ghost planes exchanged
    after every kernel over NCCL (transport="nccl", nccl_id = an NCCL unique
    id; one GPU per rank) or CUDA IPC (transport="ipc", nccl_id from
    partition.ipc_unique_id(); host-synchronised, ranks may share a GPU). State
    in the slab's local numbering (yee_slab_dofs); energy() returns this
    slab's part."""

    def __init__(self, nx, ny, nz, dx, dy, dz, dt, rank, nranks, nccl_id: bytes | None,
                 units: UnitSystem | None = None, precision: int = 8, device: int = 0,
                 transport: str = "nccl"):
        units = units or UnitSystem()
        h = C.c_void_p()
        idbuf = ((C.c_char * 128).from_buffer_copy(nccl_id.ljust(128, b"\0")[:128])
                 if nccl_id else None)
        L.check(L.lib().sfeec_yee_create_slab_transport(
            nx, ny, nz, dx, dy, dz, dt, units.eps0, units.mu0, precision, rank, nranks,
            {"nccl": 0, "ipc": 1}[transport], idbuf, device, C.byref(h)))
        self._h = h
        ne, nf = C.c_int64(), C.c_int64()
        L.check(L.lib().sfeec_yee_dof_counts(h, C.byref(ne), C.byref(nf)))
        self.n_edges, self.n_faces = ne.value, nf.value
        self.dt = dt


class YeeGroup:
    """All z-slabs of one PEC lattice on one GPU, ghosts copied on the device:
    the multi-rank step verified with a single GPU. Global PEC numbering."""

    def __init__(self, nx, ny, nz, dx, dy, dz, dt, nranks, units: UnitSystem | None = None,
                 precision: int = 8, device: int = 0):
        units = units or UnitSystem()
        h = C.c_void_p()
        L.check(L.lib().sfeec_yee_group_create(nx, ny, nz, dx, dy, dz, dt, units.eps0,
                                               units.mu0, precision, nranks, device,
                                               C.byref(h)))
        self._h = h
        c, _ = yee_operators(nx, ny, nz, dx, dy, dz)
        self.n_edges, self.n_faces = c.cols, c.rows

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and callable(getattr(L, "lib", None)):  # (module globals go at shutdown)
            L.lib().sfeec_yee_group_destroy(h)
            self._h = None

    def set_variant(self, v):
        L.check(L.lib().sfeec_yee_group_set_variant(self._h, v))

    def load(self, b, e):
        b = np.ascontiguousarray(b, np.float64)
        e = np.ascontiguousarray(e, np.float64)
        L.check(L.lib().sfeec_yee_group_set_state(self._h, L.dptr(b), L.dptr(e)))

    def fetch(self):
        b, e = np.zeros(self.n_faces), np.zeros(self.n_edges)
        L.check(L.lib().sfeec_yee_group_get_state(self._h, L.dptr(b), L.dptr(e)))
        return b, e

    def advance(self, n):
        L.check(L.lib().sfeec_yee_group_advance(self._h, int(n)))

    def energy(self):
        out = C.c_double()
        L.check(L.lib().sfeec_yee_group_energy(self._h, C.byref(out)))
        return out.value


def yee_operators(nx, ny, nz, dx, dy, dz, bc=L.BC_PEC):
    """(C, D) of the lumped Yee system in the sfeec_yee numbering (host builder)."""
    c, d = L.sfeec_csr_owned(), L.sfeec_csr_owned()
    L.check(L.lib().sfeec_build_yee_curl(nx, ny, nz, dx, dy, dz, bc, C.byref(c), C.byref(d)))
    return SparseOperator._from_owned(c), SparseOperator._from_owned(d)


def yee_masses(nx, ny, nz, dx, dy, dz, bc=L.BC_PEC):
    """(M1, M2): the consistent Q1- mass matrices of the lattice (reference
    mass_matrix, operators.cpp:133-179), same numbering as yee_operators."""
    out = []
    for form in (1, 2):
        m = L.sfeec_csr_owned()
        L.check(L.lib().sfeec_build_yee_mass(nx, ny, nz, dx, dy, dz, bc, form, C.byref(m)))
        out.append(SparseOperator._from_owned(m, True))
    return tuple(out)


class TetMesh:
    """Jittered Kuhn/Freudenthal tet mesh of the unit cube, PEC walls, first-
    order Whitney forms (host C++ builder; numbering contract in DESIGN.md)."""

    def __init__(self, n: int, jitter: float = 0.1, seed: int = 0, nzg: int | None = None,
                 planes: tuple[int, int] | None = None):
        """n^3 cubes of the unit cube; or, with nzg / planes, vertex planes
        [k0, k1] of the n x n x nzg mesh (a z-slab: the whole mesh's jitter,
        entity order and PEC walls; its cut planes are not walls)."""
        h = C.c_void_p()
        if nzg is None and planes is None:
            L.check(L.lib().sfeec_tetmesh_create(int(n), float(jitter), int(seed), C.byref(h)))
        else:
            nzg = n if nzg is None else int(nzg)
            k0, k1 = planes if planes is not None else (0, nzg)
            L.check(L.lib().sfeec_tetmesh_create_slab(int(n), nzg, int(k0), int(k1), float(jitter),
                                                      int(seed), C.byref(h)))
        self._h = h
        self.n = n
        c = [C.c_int64() for _ in range(4)]
        L.check(L.lib().sfeec_tetmesh_counts(h, *[C.byref(x) for x in c]))
        self.n_vertices, self.n_edges, self.n_faces, self.n_tets = (x.value for x in c)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and callable(getattr(L, "lib", None)):  # (module globals go at shutdown)
            L.lib().sfeec_tetmesh_destroy(h)
            self._h = None

    def geometry(self, faces: bool = True, tets: bool = True):
        """(xyz[nv,3], edge_vertices[N1,2], face_vertices[N2,3], tet_vertices[T,4]);
        faces/tets=False skip those arrays (None)."""
        xyz = np.zeros((self.n_vertices, 3))
        ev = np.zeros((self.n_edges, 2), np.int64)
        fv = np.zeros((self.n_faces, 3), np.int64) if faces else None
        tv = np.zeros((self.n_tets, 4), np.int64) if tets else None
        L.check(L.lib().sfeec_tetmesh_geometry(self._h, L.dptr(xyz), L.i64ptr(ev),
                                               L.i64ptr(fv) if faces else None,
                                               L.i64ptr(tv) if tets else None))
        return xyz, ev, fv, tv

    def pulse(self, seed: int, sigma: float = 0.1, npulses: int = 1, e0: int = 0,
              e1: int | None = None) -> np.ndarray:
        """Gaussian-pulse potential on DOF edges [e0, e1) (host C++, OpenMP):
        the same sum as inputs.pulse_one_form, without the geometry arrays."""
        from .inputs import pulse_params
        e1 = self.n_edges if e1 is None else int(e1)
        pp = pulse_params(seed, npulses)
        x0 = np.ascontiguousarray([x for x, _ in pp], np.float64).reshape(-1)
        pv = np.ascontiguousarray([q for _, q in pp], np.float64).reshape(-1)
        out = np.zeros(max(e1 - int(e0), 0))
        L.check(L.lib().sfeec_tetmesh_pulse(self._h, int(npulses), L.dptr(x0), L.dptr(pv),
                                            float(sigma), int(e0), e1, L.dptr(out)))
        return out

    def project_cavity(self, mode: int = 1) -> np.ndarray:
        """Canonical projection of A_m = sin(m pi y) sin(m pi z) dx (integral
        DOFs on the DOF edges; the PEC cube's TE cavity potential)."""
        out = np.zeros(self.n_edges)
        L.check(L.lib().sfeec_tetmesh_project_cavity(self._h, int(mode), L.dptr(out)))
        return out

    def l2_error(self, w: np.ndarray, kind: int = 1, mode: int = 1, device: int = 0):
        """(absolute, relative) L^2 error of the Whitney 1-form with DOFs w
        against A_m (kind 0) or curl curl A_m (kind 1), on the device
        (reference operators.cpp:181-257)."""
        w = np.ascontiguousarray(w, np.float64)
        if w.size != self.n_edges:
            raise InvalidParameter("l2_error: cochain length mismatch")
        out = np.zeros(2)
        L.check(L.lib().sfeec_tet_l2_error(self._h, L.dptr(w), int(kind), int(mode), device,
                                           L.dptr(out)))
        return float(out[0]), float(out[1])

    def _op(self, which, symmetric=False) -> SparseOperator:
        out = L.sfeec_csr_owned()
        L.check(L.lib().sfeec_tetmesh_operator(self._h, which, C.byref(out)))
        return SparseOperator._from_owned(out, symmetric)

    def curl(self) -> SparseOperator:
        return self._op(0)

    def mass1(self) -> SparseOperator:
        return self._op(1, True)

    def mass2(self) -> SparseOperator:
        return self._op(2, True)

    def div(self) -> SparseOperator:
        return self._op(3)

    # ---- second order (P2^-, BASELINE config 4) ----
    def p2_counts(self) -> tuple[int, int, int]:
        """(N1, N2, N3) of the P2^- 1-, 2- and 3-form spaces (PEC)."""
        c = [C.c_int64() for _ in range(3)]
        L.check(L.lib().sfeec_tetmesh_p2_counts(self._h, *[C.byref(x) for x in c]))
        return tuple(x.value for x in c)

    def p2_operator(self, which: str) -> SparseOperator:
        """'c' (N2 x N1), 'm1', 'm2' or 'd' (N3 x N2) of the P2^- system."""
        k = {"c": 0, "m1": 1, "m2": 2, "d": 3}[which]
        out = L.sfeec_csr_owned()
        L.check(L.lib().sfeec_tetmesh_p2_operator(self._h, k, C.byref(out)))
        return SparseOperator._from_owned(out, which in ("m1", "m2"))

    def p2_dofs(self, form: int):
        """(entity id, kind | slot << 1) per P2^- DOF of form 1 or 2."""
        n = self.p2_counts()[form - 1]
        ent, ks = np.zeros(n, np.int64), np.zeros(n, np.int8)
        L.check(L.lib().sfeec_tetmesh_p2_dofs(self._h, form, L.i64ptr(ent),
                                              ks.ctypes.data_as(C.POINTER(C.c_int8))))
        return ent, ks


def tet_device_scheme(n: int, jitter: float = 0.1, seed: int = 0, dt: float = 1.0,
                      kind: SplitKind = SplitKind.Strang, units: UnitSystem | None = None,
                      with_div: bool = True, warn_cfl: bool = False, layout: str = "device",
                      device: int = 0) -> "SplitScheme":
    """First-order S(M1) tet system assembled on the B200 (C, D, M1, M2, SPAI,
    Q_sym), wrapped as a (b, e) SplitScheme. Operators stay in HBM.
    layout: "device" (default: for n >= 48 advance() runs on the Kuhn-lattice
    layout -- per-vertex coefficient arrays, no index streams (DESIGN.md
    3.4); below, and for the other entry points, sliced/ELL operators built
    on the GPU), "lattice" (the lattice step at any n), "sell" (sliced/ELL
    kernels for the step too) or "host" (generic sliced/ELL layouts built
    through the host). "table": the step on the table-driven lattice (the
    layout of the second-order system) as a cross-check."""
    units = units or UnitSystem()
    h = C.c_void_p()
    counts = np.zeros(3, np.int64)
    flags = 0 if warn_cfl else L.NO_CFL_WARN
    if layout == "host":
        flags |= 8  # SFEEC_TET_HOST_LAYOUT
    elif layout == "sell":
        flags |= 32  # SFEEC_TET_NO_LATTICE
    elif layout == "lattice":
        flags |= 64  # SFEEC_TET_LATTICE
    elif layout == "table":
        flags |= 128  # SFEEC_TET_TABLE_LATTICE
    elif layout != "device":
        raise InvalidParameter("layout must be 'device', 'lattice', 'table', 'sell' or 'host'")
    L.check(L.lib().sfeec_tet_dev_create(int(n), float(jitter), int(seed), float(dt), units.eps0,
                                         units.mu0, int(SplitKind(kind)), device, flags,
                                         1 if with_div else 0, C.byref(h), L.i64ptr(counts)))
    s = SplitScheme.__new__(SplitScheme)
    s._h = h
    s._kind, s._dt, s._units = SplitKind(kind), float(dt), units
    s._formulation = Formulation.BE
    s._c = s._m2 = None
    s._n1, s._n2 = int(counts[0]), int(counts[1])
    s.n_tets = int(counts[2])
    return s


def tet_device_operators(n: int, jitter: float = 0.1, seed: int = 0, device: int = 0) -> dict:
    """Device-assembled C, M2, D, Q_sym and C^T, downloaded (parity tests)."""
    outs = [L.sfeec_csr_owned() for _ in range(5)]
    L.check(L.lib().sfeec_tet_dev_operators(int(n), float(jitter), int(seed), device,
                                            *[C.byref(o) for o in outs]))
    names = ("c", "m2", "d", "q_sym", "ct")
    return {k: SparseOperator._from_owned(o, k in ("m2", "q_sym")) for k, o in zip(names, outs)}


def p2_device_scheme(n: int, jitter: float = 0.1, seed: int = 0, dt: float = 1.0,
                     kind: SplitKind = SplitKind.Strang, units: UnitSystem | None = None,
                     with_div: bool = True, warn_cfl: bool = False, layout: str = "device",
                     device: int = 0) -> "SplitScheme":
    """Second-order P2^- system with the S(M1^2) SPAI (BASELINE config 4):
    C, M1, M2, D from the host builders; S(M1^2), SPAI, Q_sym and C^T on the
    B200; wrapped as a (b, e) SplitScheme. layout: "device" (default: for
    n >= 12 advance() runs on the table-driven Kuhn lattice, DESIGN.md 3.6 --
    Q_sym / M2 as per-vertex coefficient arrays with each symmetric pair
    stored once, C / C^T as stencil constants; sliced / ELL kernels below and
    for every other entry point), "lattice" (the lattice step from n >= 6) or
    "sell" (sliced / ELL kernels for the step too)."""
    units = units or UnitSystem()
    h = C.c_void_p()
    counts = np.zeros(5, np.int64)
    flags = 0 if warn_cfl else L.NO_CFL_WARN
    if layout == "sell":
        flags |= 32  # SFEEC_TET_NO_LATTICE
    elif layout == "lattice":
        flags |= 64  # SFEEC_TET_LATTICE
    elif layout != "device":
        raise InvalidParameter("layout must be 'device', 'lattice' or 'sell'")
    L.check(L.lib().sfeec_p2_dev_create(int(n), float(jitter), int(seed), float(dt), units.eps0,
                                        units.mu0, int(SplitKind(kind)), device, flags,
                                        1 if with_div else 0, C.byref(h), L.i64ptr(counts)))
    s = SplitScheme.__new__(SplitScheme)
    s._h = h
    s._kind, s._dt, s._units = SplitKind(kind), float(dt), units
    s._formulation = Formulation.BE
    s._c = s._m2 = None
    s._n1, s._n2 = int(counts[0]), int(counts[1])
    s.n3, s.nnz_q = int(counts[2]), int(counts[3])
    return s


def p2_device_operators(n: int, jitter: float = 0.1, seed: int = 0, device: int = 0) -> dict:
    """Device-built config-4 C, M2, D, Q_sym and C^T, downloaded (parity tests)."""
    outs = [L.sfeec_csr_owned() for _ in range(5)]
    L.check(L.lib().sfeec_p2_dev_operators(int(n), float(jitter), int(seed), device,
                                           *[C.byref(o) for o in outs]))
    names = ("c", "m2", "d", "q_sym", "ct")
    return {k: SparseOperator._from_owned(o, k in ("m2", "q_sym")) for k, o in zip(names, outs)}


def spai_device(m: SparseOperator, device: int = 0):
    """S(M1^2) SPAI of m on the GPU -> (Q by rows, fallback columns)."""
    out = L.sfeec_csr_owned()
    fb = C.c_int64()
    v = m.view()
    L.check(L.lib().sfeec_p2_spai_device(C.byref(v), device, C.byref(out), C.byref(fb)))
    return SparseOperator._from_owned(out), fb.value


PATTERNS = {"diagonal": 0, "m1": 1, "m1sq": 2}


def make_pattern(m: SparseOperator, kind: str = "m1") -> SparseOperator:
    """spai.cpp:31-72; returns the pattern as a CSR with unit values."""
    out = L.sfeec_csr_owned()
    v = m.view()
    L.check(L.lib().sfeec_make_pattern(C.byref(v), PATTERNS[kind], C.byref(out)))
    return SparseOperator._from_owned(out)


def spai_approximate_inverse(m: SparseOperator, kind: str = "m1"):
    """spai.cpp:127-286 -> (Q, report dict)."""
    out = L.sfeec_csr_owned()
    rep = np.zeros(4)
    v = m.view()
    L.check(L.lib().sfeec_spai(C.byref(v), PATTERNS[kind], C.byref(out), L.dptr(rep)))
    q = SparseOperator._from_owned(out)
    return q, {"frobenius_residual": rep[0], "avg_nnz_per_row": rep[1],
               "max_column_residual": rep[2], "fallback_columns": int(rep[3])}


def device_count() -> int:
    return int(L.lib().sfeec_device_count())
