"""z-slab partition of the unstructured (tet) leapfrog.

The tet DOF numbering is k-major: entities whose base vertex
lies in vertex planes [P_r, P_{r+1}) form one contiguous id range. Rank r owns
that range; its local vectors cover planes [P_r - 1, P_{r+1}] (a one-plane
halo each side -- every operator row of an owned entity only references
entities within one plane: the first-order one-layer halo). Local operators
are row slices with columns shifted by the local start: no renumbering.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .scheme import SparseOperator, symmetric_part, transpose


def plane_splits(n: int, nranks: int) -> np.ndarray:
    """Vertex-plane boundaries P_0 = 0 < ... < P_R = n + 1 (balanced)."""
    if not 1 <= nranks <= n + 1:
        raise ValueError("need 1 <= nranks <= n + 1")
    return np.array([(r * (n + 1)) // nranks for r in range(nranks + 1)])


def entity_plane_offsets(base_vertices: np.ndarray, n: int) -> np.ndarray:
    """off[k] = first id whose base vertex is in plane k (k = 0..n+1)."""
    planes = base_vertices // ((n + 1) * (n + 1))
    if np.any(np.diff(planes) < 0):
        raise ValueError("numbering is not k-major")
    return np.searchsorted(planes, np.arange(n + 2), side="left")


@dataclass
class LocalSystem:
    rank: int
    nranks: int
    q: SparseOperator   # Q_sym, owned edges x local edges
    ct: SparseOperator  # C^T, owned edges x local faces
    c: SparseOperator   # C, owned faces x local edges
    m2: SparseOperator  # M2, owned faces x local faces
    edge_range: np.ndarray  # len, own_lo, own_hi, first_len, last_len (local indices)
    face_range: np.ndarray
    edge_global: tuple  # (global start of the local range, owned global lo, hi)
    face_global: tuple


def _rows(a: SparseOperator, lo: int, hi: int, col0: int, ncols: int) -> SparseOperator:
    rp = a.row_ptr[lo:hi + 1] - a.row_ptr[lo]
    sl = slice(int(a.row_ptr[lo]), int(a.row_ptr[hi]))
    ci = a.col_idx[sl].astype(np.int64) - col0
    if ci.size and (ci.min() < 0 or ci.max() >= ncols):
        raise ValueError("operator row references entities beyond the one-plane halo")
    return SparseOperator(hi - lo, ncols, rp, ci.astype(np.int32), a.val[sl].copy())


def slab_system(sys_, rank: int, nranks: int, q_sym: SparseOperator | None = None,
                ct: SparseOperator | None = None, halo: int = 1,
                bases: tuple | None = None) -> LocalSystem:
    """Local operators of rank `rank` (sys_ has .mesh, .q, .c, .m2). halo =
    vertex planes each side (1 first order, 2 for config 4's S(M1^2) Q);
    bases = (base vertex per 1-form DOF, per 2-form DOF), default the
    first-order edges / faces."""
    n = sys_.mesh.n
    if bases is None:
        _, ev, fv, _ = sys_.mesh.geometry()
        bases = (ev[:, 0], fv[:, 0])
    P = plane_splits(n, nranks)
    if np.any(np.diff(P) < halo):
        raise ValueError("every rank must own at least `halo` vertex planes")
    q_sym = q_sym if q_sym is not None else symmetric_part(sys_.q)
    ct = ct if ct is not None else transpose(sys_.c)
    out = {}
    for kind, base in (("e", bases[0]), ("f", bases[1])):
        off = entity_plane_offsets(base, n)
        p0, p1 = P[rank], P[rank + 1]
        g_lo = off[max(p0 - halo, 0)]
        g_hi = off[min(p1 + halo, n + 1)]
        o_lo, o_hi = off[p0], off[p1]
        first = off[p0 + halo] - off[p0]
        last = off[p1] - off[p1 - halo]
        rng = np.array([g_hi - g_lo, o_lo - g_lo, o_hi - g_lo, first, last], np.int64)
        out[kind] = (rng, (int(g_lo), int(o_lo), int(o_hi)))
    (er, eg), (fr, fg) = out["e"], out["f"]
    return LocalSystem(
        rank, nranks,
        q=_rows(q_sym, eg[1], eg[2], eg[0], int(er[0])),
        ct=_rows(ct, eg[1], eg[2], fg[0], int(fr[0])),
        c=_rows(sys_.c, fg[1], fg[2], eg[0], int(er[0])),
        m2=_rows(sys_.m2, fg[1], fg[2], fg[0], int(fr[0])),
        edge_range=er, face_range=fr, edge_global=eg, face_global=fg)


@dataclass
class SlabInfo:
    """Ranges of a device-built slab (sfeec_part_create_tet info)."""
    rank: int
    nranks: int
    n1: int
    n2: int
    edge_range: np.ndarray
    face_range: np.ndarray
    edge_global: tuple
    face_global: tuple
    dt: float


class TetPart:
    """One rank's partitioned device leapfrog (sfeec_part)."""

    KERNEL_CLASSES = ("K-Q", "K-Cb", "K-CTe", "K-M2", "exchange")

    def __init__(self, ls: LocalSystem, dt: float, eps0=1.0, mu0=1.0, nccl_id: bytes | None = None,
                 device: int = 0):
        h = C.c_void_p()
        views = [ls.q.view(), ls.c.view(), ls.ct.view(), ls.m2.view()]
        self._keep = (ls, views)
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        L.check(L.lib().sfeec_part_create(*[C.byref(v) for v in views],
                                          L.i64ptr(ls.edge_range), L.i64ptr(ls.face_range),
                                          float(dt), eps0, mu0, ls.rank, ls.nranks, idbuf,
                                          device, C.byref(h)))
        self._h = h
        self.ls = ls

    @classmethod
    def from_device(cls, n: int, jitter: float, seed: int, rank: int, nranks: int,
                    dt: float = 0.0, eps0=1.0, mu0=1.0, nccl_id: bytes | None = None,
                    device: int = 0, order: int = 1) -> "TetPart":
        """Rank `rank`'s slab of the tet system, assembled and row-sliced on
        its own device (no host CSR): order 1 = configs 1/3/5 (P1-, S(M1),
        one-plane halo), order 2 = config 4 (P2-, S(M1^2), two-plane halo).
        dt <= 0: 0.5 x the CFL estimate of the full operators (bitwise
        configs.cfl_dt of the single-GPU device scheme)."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        info = np.zeros(19, np.int64)
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        fn = L.lib().sfeec_part_create_tet if order == 1 else L.lib().sfeec_part_create_p2
        L.check(fn(int(n), float(jitter), int(seed), float(dt), eps0, mu0, int(rank), int(nranks),
                   idbuf, int(device), C.byref(h), L.i64ptr(info)))
        self._h = h
        self._keep = None
        self.ls = SlabInfo(rank, nranks, int(info[0]), int(info[1]), info[2:7].copy(),
                           info[7:12].copy(), tuple(int(x) for x in info[12:15]),
                           tuple(int(x) for x in info[15:18]),
                           float(info[18:19].view(np.float64)[0]))
        return self

    @property
    def dt(self) -> float:
        return self.ls.dt

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and callable(getattr(L, "lib", None)):  # (module globals go at shutdown)
            L.lib().sfeec_part_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def attach_ipc(self, comm_id: bytes) -> None:
        """Collective: the host-synchronised CUDA-IPC halo transport for a
        multi-rank handle created without an NCCL id (comm_id from
        ipc_unique_id(); the ranks may share a GPU)."""
        idbuf = (C.c_char * 128).from_buffer_copy(comm_id.ljust(128, b"\0")[:128])
        L.check(L.lib().sfeec_part_attach_ipc(self._h, C.cast(idbuf, C.c_void_p)))

    def load_global(self, b, e, time=0.0):
        eg, fg = self.ls.edge_global, self.ls.face_global
        bo = np.ascontiguousarray(b[fg[1]:fg[2]], np.float64)
        eo = np.ascontiguousarray(e[eg[1]:eg[2]], np.float64)
        L.check(L.lib().sfeec_part_set_state(self._h, L.dptr(bo), L.dptr(eo), time))

    def fetch_into(self, b, e):
        eg, fg = self.ls.edge_global, self.ls.face_global
        bo, eo, t = np.zeros(fg[2] - fg[1]), np.zeros(eg[2] - eg[1]), C.c_double()
        L.check(L.lib().sfeec_part_get_state(self._h, L.dptr(bo), L.dptr(eo), C.byref(t)))
        b[fg[1]:fg[2]] = bo
        e[eg[1]:eg[2]] = eo
        return t.value

    def advance(self, n):
        L.check(L.lib().sfeec_part_advance(self._h, int(n)))

    def energy(self):
        out = C.c_double()
        L.check(L.lib().sfeec_part_energy(self._h, C.byref(out)))
        return out.value

    def apply(self, which: str, x_local: np.ndarray) -> np.ndarray:
        """Owned rows of A x for a local-range x (A in q, c, ct, m2)."""
        k = {"q": 0, "c": 1, "ct": 2, "m2": 3}[which]
        er, fr = self.ls.edge_range, self.ls.face_range
        ncols = int(er[0] if which in ("q", "c") else fr[0])
        nrows = int(er[2] - er[1] if which in ("q", "ct") else fr[2] - fr[1])
        x = np.ascontiguousarray(x_local, np.float64)
        if x.shape != (ncols,):
            raise ValueError(f"apply({which}): x must have {ncols} entries")
        y = np.zeros(nrows)
        L.check(L.lib().sfeec_part_apply(self._h, k, L.dptr(x), L.dptr(y)))
        return y

    def device_ptrs(self):
        """(b_local, e_local, stream) device addresses."""
        b, e, s = C.c_void_p(), C.c_void_p(), C.c_void_p()
        L.check(L.lib().sfeec_part_device_ptrs(self._h, C.byref(b), C.byref(e), C.byref(s)))
        return b.value, e.value, s.value

    def last_launches(self) -> int:
        return int(L.lib().sfeec_part_last_launches(self._h))

    def step_bytes(self) -> float:
        return float(L.lib().sfeec_part_step_bytes(self._h))

    def kernel_timing(self, enable: bool = True) -> dict:
        """Per-class device time since the last call (then (dis)arm timing)."""
        ms, n, by = np.zeros(5), np.zeros(5, np.int64), np.zeros(5)
        L.check(L.lib().sfeec_part_kernel_timing(self._h, 1 if enable else 0, L.dptr(ms),
                                                 L.i64ptr(n), L.dptr(by)))
        return {k: {"ms": ms[i], "launches": int(n[i]), "bytes_per_launch": by[i]}
                for i, k in enumerate(self.KERNEL_CLASSES)}


def advance_local(parts: list[TetPart], n: int) -> None:
    arr = (C.c_void_p * len(parts))(*[p.handle for p in parts])
    L.check(L.lib().sfeec_part_advance_local(arr, len(parts), int(n)))


def energy_local(parts: list[TetPart]) -> float:
    arr = (C.c_void_p * len(parts))(*[p.handle for p in parts])
    out = C.c_double()
    L.check(L.lib().sfeec_part_energy_local(arr, len(parts), C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# Kuhn-lattice slabs (lattice_slab.cu): the multi-rank production path
# ---------------------------------------------------------------------------
def ipc_unique_id() -> bytes:
    """A fresh id for the CUDA-IPC transport (broadcast it to every rank)."""
    buf = (C.c_char * 128)()
    L.check(L.lib().sfeec_ipc_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


class LatticeSlab:
    """Rank `rank` of `nranks` of the first-order leapfrog on the Kuhn lattice,
    split into z-slabs of whole vertex planes (lattice_slab.cu). Each rank
    assembles only its own slab of the n x n x nzg mesh (nzg = n: the unit
    cube; nzg = n * nranks: a weak-scaling stack of n^3 blocks). State vectors
    are the rank's owned DOFs, a contiguous range of the whole mesh's
    k-major numbering (edges [e_glob, e_glob + n1), faces [f_glob, f_glob + n2)).
    transport: "nccl" (comm_id = an NCCL unique id; one GPU per rank) or "ipc"
    (comm_id from ipc_unique_id(); host-synchronised, ranks may share a GPU).
    energy(), cfl_number() and curl() are collective."""

    def __init__(self, n: int, jitter: float = 0.1, seed: int = 0, nzg: int | None = None,
                 dt: float = 1.0, rank: int = 0, nranks: int = 1, transport: str = "nccl",
                 comm_id: bytes | None = None, kind: int = 1, eps0: float = 1.0,
                 mu0: float = 1.0, device: int = 0):
        self.n, self.nzg = int(n), int(nzg if nzg is not None else n)
        self.jitter, self.seed = float(jitter), int(seed)
        self.rank, self.nranks = int(rank), int(nranks)
        tr = {"nccl": 0, "ipc": 1}[transport]
        idbuf = None
        if comm_id is not None:
            idbuf = (C.c_char * 128).from_buffer_copy(comm_id.ljust(128, b"\0")[:128])
        h = C.c_void_p()
        info = np.zeros(10, np.int64)
        L.check(L.lib().sfeec_lslab_create(self.n, self.nzg, self.jitter, self.seed, float(dt),
                                           float(eps0), float(mu0), int(kind), self.rank,
                                           self.nranks, tr,
                                           C.cast(idbuf, C.c_void_p) if idbuf else None,
                                           int(device), C.byref(h), L.i64ptr(info)))
        self._h = h
        self.n1, self.n2 = int(info[0]), int(info[1])
        self.e_glob, self.f_glob = int(info[2]), int(info[3])
        self.planes = (int(info[4]), int(info[5]))
        self.assembled = (int(info[6]), int(info[7]))
        self.e_local0, self.f_local0 = int(info[8]), int(info[9])
        self._dt = float(dt)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and callable(getattr(L, "lib", None)):
            L.lib().sfeec_lslab_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def mesh(self):
        """the host TetMesh of this rank's assembled slab (ids = slab-local)"""
        from .scheme import TetMesh
        return TetMesh(self.n, self.jitter, self.seed, nzg=self.nzg, planes=self.assembled)

    def pulse(self, seed: int, sigma: float = 0.1, npulses: int = 1) -> np.ndarray:
        """the Gaussian-pulse potential on the owned edges"""
        return self.mesh().pulse(seed, sigma, npulses, self.e_local0, self.e_local0 + self.n1)

    def set_state(self, b: np.ndarray, e: np.ndarray, time: float = 0.0) -> None:
        b = np.ascontiguousarray(b, np.float64)
        e = np.ascontiguousarray(e, np.float64)
        if b.size != self.n2 or e.size != self.n1:
            raise L.InvalidParameter("lattice slab: state sizes differ from the owned DOFs")
        L.check(L.lib().sfeec_lslab_set_state(self._h, L.dptr(b), L.dptr(e), float(time)))

    def get_state(self):
        b, e, t = np.zeros(self.n2), np.zeros(self.n1), C.c_double()
        L.check(L.lib().sfeec_lslab_get_state(self._h, L.dptr(b), L.dptr(e), C.byref(t)))
        return b, e, t.value

    def advance(self, nsteps: int) -> None:
        L.check(L.lib().sfeec_lslab_advance(self._h, int(nsteps)))

    def energy(self) -> float:
        out = C.c_double()
        L.check(L.lib().sfeec_lslab_energy(self._h, C.byref(out)))
        return out.value

    def cfl_number(self) -> float:
        out = C.c_double()
        L.check(L.lib().sfeec_lslab_cfl_number(self._h, C.byref(out)))
        return out.value

    def set_dt(self, dt: float) -> None:
        L.check(L.lib().sfeec_lslab_set_dt(self._h, float(dt)))
        self._dt = float(dt)

    def dt(self) -> float:
        return self._dt

    def curl(self, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float64)
        if a.size != self.n1:
            raise L.InvalidParameter("lattice slab: a must hold the owned edges")
        b = np.zeros(self.n2)
        L.check(L.lib().sfeec_lslab_curl(self._h, L.dptr(a), L.dptr(b)))
        return b

    def stream_ptr(self) -> int:
        s = C.c_void_p()
        L.check(L.lib().sfeec_lslab_stream(self._h, C.byref(s)))
        return s.value or 0

    def last_launches(self) -> int:
        return int(L.lib().sfeec_lslab_last_launches(self._h))

    def step_bytes(self) -> float:
        return float(L.lib().sfeec_lslab_step_bytes(self._h))

    KERNEL_CLASSES = ("K-Q", "K-Cb", "K-CTe", "K-M2")

    def kernel_timing(self, enable: bool = True) -> dict:
        ms, n, by = np.zeros(4), np.zeros(4, np.int64), np.zeros(4)
        L.check(L.lib().sfeec_lslab_kernel_timing(self._h, 1 if enable else 0, L.dptr(ms),
                                                  L.i64ptr(n), L.dptr(by)))
        return {k: {"ms": ms[i], "launches": int(n[i]), "bytes_per_launch": by[i]}
                for i, k in enumerate(self.KERNEL_CLASSES)}
