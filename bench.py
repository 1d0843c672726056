#!/usr/bin/env python
"""Benchmark of the B200 SFEEC leapfrog (BASELINE.json metric:
"edge+face DOF-updates/sec per leapfrog step; achieved HBM GB/s vs peak").

Default workload = BASELINE.json configs[4], the largest single-GPU config:
256^3 cubes x 6 Kuhn tets (100.7M tets), jitter 0.1h, first-order Whitney
forms, S(M1) SPAI, PEC walls, 8 seeded Gaussian pulses in A, B0 = C A, E0 = 0,
dt = 0.5 CFL, fp64. A "step" is one leapfrog step over all N1 + N2 DOFs
(318.6M).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config tet256|tet128|tet16|yee256|yee256_f32|p2_64|...]

Other configs: tet16 = configs[0] (16^3 x 6 tets, S(M1) SPAI, jitter 0.1),
yee256 = configs[1] (Yee/lumped-mass 256^3, PEC, Courant 0.5), tet128 =
configs[2] (128^3 x 6 tets, jitter 0.15, Gaussian pulse), p2_64 = configs[3].
Under torchrun (N > 1) the Yee configs run one 256^3 block per rank stacked in
z (weak scaling); the tet configs split the one mesh into N z-slabs (strong
scaling).
`--impl reference` times the reference CPU step (oracle/_ref: the unmodified
reference SplitScheme::step, dynamics.cpp:69-90) on the host cores, on
operators built without the product library (_ref_operators).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edge+face DOF-updates/sec per leapfrog step; achieved HBM GB/s vs peak"
UNIT = "DOF-updates/s"

CONFIGS = {
    "yee256": dict(kind="yee", n=256, precision=8, dtype="f64", ref_n=256,
                   desc="BASELINE configs[1] Yee/lumped-mass SFEEC, 256^3 cells, PEC, "
                        "Courant 0.5"),
    "yee256_f32": dict(kind="yee", n=256, precision=4, dtype="f32", ref_n=256,
                       desc="BASELINE configs[1] Yee/lumped-mass SFEEC in fp32, 256^3 cells, "
                            "PEC, Courant 0.5"),
    "tet16": dict(kind="tet", n=16, jitter=0.1, init="gaussian", dtype="f64", ref_n=16,
                  desc="BASELINE configs[0]: 16^3 x 6 Kuhn tets, jitter 0.1h, P1-, S(M1) "
                       "SPAI, PEC, dt = 0.5 CFL"),
    "tet64": dict(kind="tet", n=64, jitter=0.15, init="pulse", dtype="f64", ref_n=64,
                  desc="64^3 x 6 Kuhn tets, jitter 0.15h, P1-, S(M1) SPAI, PEC, pulse"),
    "tet128": dict(kind="tet", n=128, jitter=0.15, init="pulse", dtype="f64", ref_n=128,
                   desc="BASELINE configs[2]: 128^3 x 6 Kuhn tets, jitter 0.15h, P1-, S(M1) "
                        "SPAI, PEC, Gaussian pulse width 0.1, dt = 0.5 CFL"),
    "p2_64": dict(kind="p2", n=64, jitter=0.1, init="gaussian", dtype="f64", ref_n=3,
                  desc="BASELINE configs[3]: 64^3 x 6 Kuhn tets, jitter 0.1h, P2-, S(M1^2) "
                       "(2-ring) SPAI, PEC, dt = 0.5 CFL"),
    "p2_32": dict(kind="p2", n=32, jitter=0.1, init="gaussian", dtype="f64", ref_n=3,
                  desc="32^3 x 6 Kuhn tets, jitter 0.1h, P2-, S(M1^2) SPAI, PEC (smaller "
                       "config-4 system)"),
    "tet256": dict(kind="tet", n=256, jitter=0.1, init="pulse", npulses=8, dtype="f64", ref_n=128,
                   desc="BASELINE configs[4]: 256^3 x 6 Kuhn tets (100.7M tets), jitter 0.1h, "
                        "P1-, S(M1) SPAI, PEC, 8 Gaussian pulses, dt = 0.5 CFL"),
}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.samples, self._stop = device, [], threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# --------------------------------------------------------------------------
# workloads
# --------------------------------------------------------------------------
def yee_setup(n, precision, device):
    """Operators + initial state of configs[1] on an n^3 unit cube."""
    import paper_2301_01753_b200 as S
    from paper_2301_01753_b200 import inputs
    h = 1.0 / n
    dt = 0.5 / (np.sqrt(3.0) * n)  # Courant 0.5: c dt sqrt(sum 1/d^2) = 0.5
    y = S.YeeScheme(n, n, n, h, h, h, dt, bc=1, precision=precision, device=device)
    a = inputs.gaussian(20260101, y.n_edges)
    # B0 = C A on the device: a b-kick with h = -dV from e = A gives b = C A (Q = I/dV)
    y.load(np.zeros(y.n_faces), a)
    y.flow_he(-(h ** 3))
    b0, _, _ = y.fetch()
    return y, b0, np.zeros(y.n_edges), dt


def yee_slab_setup(n, precision, device, rank, world, dist, transport="nccl"):
    """Rank `rank` of a 256 x 256 x (256 world) PEC lattice (weak scaling): the
    z-slab with NCCL ghost exchange; A drawn by global edge id."""
    import paper_2301_01753_b200 as S
    from paper_2301_01753_b200 import inputs
    h = 1.0 / n
    dt = 0.5 / (np.sqrt(3.0) * n)
    nz = n * world
    from paper_2301_01753_b200.partition import ipc_unique_id
    new_id = ipc_unique_id if transport == "ipc" else S.nccl_unique_id
    ids = [new_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    y = S.YeeSlab(n, n, nz, h, h, h, dt, rank, world, ids[0], precision=precision,
                  device=device, transport=transport)
    em, _ = S.yee_slab_dofs(n, n, nz, rank, world)
    a = inputs.gaussian_ids(20260101, em)
    y.load(np.zeros(y.n_faces), a)          # exchanges the ghost planes
    y.flow_he(-(h ** 3))                    # b = C A on the owned faces
    b0, _, _ = y.fetch()
    return y, b0, np.zeros(y.n_edges), dt


class YeeRunner:
    def __init__(self, cfg, device, rank=0, world=1, dist=None, transport="nccl"):
        from paper_2301_01753_b200 import _lib as L
        self.L = L
        if dist is not None:
            self.y, self.b0, self.e0, self.dt = yee_slab_setup(cfg["n"], cfg["precision"],
                                                                device, rank, world, dist,
                                                                transport)
            self.kernel_label = ("two-step fused TMA sweep per z-slab (two ghost planes) + "
                                 "NCCL ghost-plane exchange overlapped with the interior chunks")
        else:
            self.y, self.b0, self.e0, self.dt = yee_setup(cfg["n"], cfg["precision"], device)
        self.ndof = self.y.n_edges + self.y.n_faces
        self.n1, self.n2 = self.y.n_edges, self.y.n_faces
        self.prec = cfg["precision"]

    def set_stream(self, ptr):
        self.L.check(self.L.lib().sfeec_yee_set_stream(self.y.handle, ctypes.c_void_p(ptr)))

    def load(self):
        self.y.load(self.b0, self.e0)

    def advance(self, k):
        self.y.advance(k)

    def launches(self):
        return self.y.last_launches()

    def timing(self, enable):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        self.L.check(self.L.lib().sfeec_yee_kernel_timing(self.y.handle, 1 if enable else 0,
                                                           ms, n))
        return ms.value, n.value

    def dominant(self, k_steps):
        """(name, algorithmic bytes per launch, avg ms per launch) of the fused
        sweep. The timed launches cover the k_steps (e, b) pairs after the
        opening b-half-kick (the closing half-kick is folded into the last
        sweep); a two-step sweep (k_fused2_tma) advances two of them per
        launch, so its algorithmic bytes per launch are two steps' worth
        (SURVEY.md 8(d))."""
        self.timing(True)
        self.y.advance(k_steps)
        ms, n = self.timing(False)
        n = max(n, 1)
        per_launch = k_steps / n
        name = ("k_fused2_tma (two e-kick + b-kick pairs per z-sweep)" if per_launch > 1.5
                else "k_fused_tma (e-kick + b-kick sweep)")
        return name, self.y.step_bytes() * per_launch, ms / n

    def step_bytes(self):
        return self.y.step_bytes()

    def diagnostics(self):
        """(discrete energy of the device state (this slab's part), Gauss residual or None)"""
        return self.y.energy(), None

    def e2e(self, k, torch):
        L = self.L
        pin_b = torch.from_numpy(self.b0).pin_memory()
        pin_e = torch.from_numpy(self.e0).pin_memory()
        out_b, out_e = torch.empty_like(pin_b).pin_memory(), torch.empty_like(pin_e).pin_memory()
        t0 = time.perf_counter()
        L.check(L.lib().sfeec_yee_set_state(self.y.handle, dptr(pin_b), dptr(pin_e), 0.0))
        self.y.advance(k)
        L.check(L.lib().sfeec_yee_get_state(self.y.handle, dptr(out_b), dptr(out_e), None))
        return time.perf_counter() - t0

    kernel_label = ("two leapfrog steps per TMA-pipelined z-sweep, intermediates in registers + "
                    "shared memory (k_fused2_tma; SFEEC_YEE_VARIANT=2 selects the one-step "
                    "k_fused_tma)")


def tet_setup(cfg, device):
    """Mesh numbering on the host; C, D, M1, M2, SPAI and Q_sym assembled on the
    device (tet_device.cu, bitwise the host builders); dt = 0.5 CFL."""
    import paper_2301_01753_b200 as S
    from paper_2301_01753_b200 import configs, inputs
    t0 = time.perf_counter()
    if cfg["kind"] == "p2":
        # SFEEC_P2_LAYOUT=sell keeps the sliced / ELL step (A/B against the lattice)
        s = S.p2_device_scheme(cfg["n"], cfg["jitter"], seed=2023, dt=1.0, with_div=True,
                               layout=os.environ.get("SFEEC_P2_LAYOUT", "device"), device=device)
        b0 = s.apply("c", inputs.gaussian(7, s._n1))
        s.set_dt(configs.cfl_dt(s))
        return (s._n1, s._n2), s, b0, np.zeros(s._n1), time.perf_counter() - t0
    # SFEEC_TET_LAYOUT=table|sell|lattice: A/B of the step layouts (default: device)
    s = S.tet_device_scheme(cfg["n"], cfg["jitter"], seed=2023, dt=1.0, with_div=True,
                            layout=os.environ.get("SFEEC_TET_LAYOUT", "device"), device=device)
    if cfg["init"] == "gaussian":
        a = inputs.gaussian(7, s._n1)
    else:  # host C++ projection of the pulses (sfeec_tetmesh_pulse)
        a = S.TetMesh(cfg["n"], cfg["jitter"], 2023).pulse(7, 0.1, cfg.get("npulses", 1))
    b0 = s.apply("c", a)
    s.set_dt(configs.cfl_dt(s))
    setup_s = time.perf_counter() - t0
    return (s._n1, s._n2), s, b0, np.zeros(s._n1), setup_s


class TetRunner:
    def __init__(self, cfg, device):
        import paper_2301_01753_b200 as S
        from paper_2301_01753_b200 import _lib as L
        self.S, self.L = S, L
        (self.n1, self.n2), self.s, self.b0, self.e0, self.setup_s = tet_setup(cfg, device)
        if cfg["kind"] == "p2" and os.environ.get("SFEEC_P2_LAYOUT", "device") == "sell":
            self.layout = "sell"
            self.kernel_label = "SpMV chain K-M2, K-CTe, K-Q, K-Cb in sliced layouts (spmv_kernels.cu)"
        elif cfg["kind"] == "p2":  # second order: the table-driven lattice
            self.layout = "table"
            self.kernel_label = ("table-driven Kuhn-lattice K-M2, K-CTe, K-Q, K-Cb: one thread per "
                                 "(vertex, DOF type), per-vertex coefficient arrays with symmetric "
                                 "pairs stored once, C / C^T as stencil constants "
                                 "(table_lattice.cu)")
        self.ndof = self.n1 + self.n2
        self.dt = self.s.dt()

    def set_stream(self, ptr):
        self.L.check(self.L.lib().sfeec_dev_set_stream(self.s.handle, ctypes.c_void_p(ptr)))

    def load(self):
        self.s.load(self.S.make_state(self.S.Formulation.BE, self.b0, self.e0))

    def advance(self, k):
        self.L.check(self.L.lib().sfeec_dev_advance(self.s.handle, int(k)))

    def launches(self):
        return self.s.last_launches()

    def dominant(self, k_steps):
        self.s.kernel_timing(True)
        self.advance(k_steps)
        t = self.s.kernel_timing(False)
        name = max((k for k in t if k != "other"), key=lambda k: t[k]["ms"])
        self.per_kernel = {k: {"avg_ms": v["ms"] / max(v["launches"], 1),
                               "bytes_per_launch": v["bytes_per_launch"],
                               "gbs": v["bytes_per_launch"] / (v["ms"] / max(v["launches"], 1)
                                                               * 1e-3) / 1e9
                               if v["ms"] > 0 else None}
                           for k, v in t.items() if k != "other"}
        d = t[name]
        return name, d["bytes_per_launch"], d["ms"] / max(d["launches"], 1)

    def step_bytes(self):
        return self.s.step_bytes()

    def diagnostics(self):
        """energy (dynamics.cpp:92-102) and Gauss residual max|D b| (:104-112)
        of the device-resident state"""
        en, g = ctypes.c_double(), ctypes.c_double()
        self.L.check(self.L.lib().sfeec_dev_energy(self.s.handle, ctypes.byref(en)))
        self.L.check(self.L.lib().sfeec_dev_gauss_residual(self.s.handle, ctypes.byref(g)))
        return en.value, g.value

    def e2e(self, k, torch):
        L = self.L
        pin_b = torch.from_numpy(self.b0).pin_memory()
        pin_e = torch.from_numpy(self.e0).pin_memory()
        out_b, out_e = torch.empty_like(pin_b).pin_memory(), torch.empty_like(pin_e).pin_memory()
        t = ctypes.c_double()
        t0 = time.perf_counter()
        L.check(L.lib().sfeec_dev_set_state(self.s.handle, dptr(pin_b), self.n2, dptr(pin_e),
                                            self.n1, 0.0))
        self.advance(k)
        L.check(L.lib().sfeec_dev_get_state(self.s.handle, dptr(out_b), dptr(out_e),
                                            ctypes.byref(t)))
        return time.perf_counter() - t0

    kernel_label = ("Kuhn-lattice K-M2, K-CTe, K-Q, K-Cb: per-vertex stencils with per-vertex "
                    "coefficient arrays, symmetric pairs stored once, no index streams (lattice.cu)")
    layout = "lattice"


class TetSlabRunner:
    """Rank `rank` of the tet system split into z-slabs (strong scaling: the
    mesh is fixed, every rank assembles it on its own GPU and keeps its owned
    rows; partition.cu, 4 NCCL halo exchanges per step; one-plane halo for
    P1-, two-plane for config 4's S(M1^2) Q)."""

    scaling = "strong"
    layout = "sell"
    kernel_label = ("SpMV chain K-M2, K-CTe, K-Q, K-Cb over the owned rows + NCCL halo-plane "
                    "exchange before each (partition.cu)")

    def __init__(self, cfg, device, rank, world, dist, transport="nccl"):
        import paper_2301_01753_b200 as S
        from paper_2301_01753_b200 import inputs, partition
        t0 = time.perf_counter()
        ids = [None]
        ipc = transport == "ipc" and world > 1
        if dist is not None:
            new_id = partition.ipc_unique_id if ipc else S.nccl_unique_id
            ids = [new_id() if rank == 0 else None]
            dist.broadcast_object_list(ids, src=0)
        self.p = partition.TetPart.from_device(cfg["n"], cfg["jitter"], 2023, rank, world,
                                               nccl_id=None if ipc else ids[0], device=device,
                                               order=2 if cfg["kind"] == "p2" else 1)
        if ipc:
            self.p.attach_ipc(ids[0])
        ls = self.p.ls
        eg, er, fg = ls.edge_global, ls.edge_range, ls.face_global
        if cfg["init"] == "gaussian":
            a = inputs.gaussian_ids(7, np.arange(eg[0], eg[0] + er[0]))
        else:
            a = S.TetMesh(cfg["n"], cfg["jitter"], 2023).pulse(7, 0.1, cfg.get("npulses", 1),
                                                               eg[0], eg[0] + er[0])
        self.b0 = self.p.apply("c", a)                 # owned faces of C A
        self.e0 = np.zeros(eg[2] - eg[1])
        self.n1, self.n2 = ls.n1, ls.n2
        self.ndof = ls.n1 + ls.n2                       # whole job (strong scaling)
        self.dt = self.p.dt
        self.setup_s = time.perf_counter() - t0
        self._stream = None

    def stream(self, torch):
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.p.device_ptrs()[2])
        return self._stream

    def set_stream(self, ptr):
        pass  # the partition handle keeps its own stream (stream() above)

    @property
    def L(self):
        from paper_2301_01753_b200 import _lib
        return _lib

    def load(self):
        L = self.L
        L.check(L.lib().sfeec_part_set_state(self.p.handle, L.dptr(self.b0), L.dptr(self.e0), 0.0))

    def advance(self, k):
        self.p.advance(k)

    def launches(self):
        return self.p.last_launches()

    def dominant(self, k_steps):
        self.p.kernel_timing(True)
        self.advance(k_steps)
        t = self.p.kernel_timing(False)
        self.per_kernel = {k: {"avg_ms": v["ms"] / max(v["launches"], 1),
                               "launches": v["launches"],
                               "bytes_per_launch": v["bytes_per_launch"],
                               "gbs": v["bytes_per_launch"] / (v["ms"] / max(v["launches"], 1)
                                                               * 1e-3) / 1e9
                               if v["ms"] > 0 and v["bytes_per_launch"] > 0 else None}
                           for k, v in t.items()}
        name = max(("K-Q", "K-Cb", "K-CTe", "K-M2"), key=lambda k: t[k]["ms"])
        d = t[name]
        return name, d["bytes_per_launch"], d["ms"] / max(d["launches"], 1)

    def step_bytes(self):
        return self.p.step_bytes()

    def diagnostics(self):
        return self.p.energy(), None  # this rank's part (summed over ranks by the caller)

    def e2e(self, k, torch):
        L = self.L
        pin_b = torch.from_numpy(self.b0).pin_memory()
        pin_e = torch.from_numpy(self.e0).pin_memory()
        out_b, out_e = torch.empty_like(pin_b).pin_memory(), torch.empty_like(pin_e).pin_memory()
        t0 = time.perf_counter()
        L.check(L.lib().sfeec_part_set_state(self.p.handle, dptr(pin_b), dptr(pin_e), 0.0))
        self.advance(k)
        L.check(L.lib().sfeec_part_get_state(self.p.handle, dptr(out_b), dptr(out_e), None))
        self.e2e_bytes = 8 * (self.b0.size + self.e0.size)
        return time.perf_counter() - t0


class LatSlabRunner:
    """Rank `rank` of the first-order tet leapfrog on Kuhn-lattice z-slabs
    (lattice_slab.cu): every rank assembles only its slab on its own GPU and
    exchanges one-plane ghosts over NCCL after each kernel. Weak scaling
    (default): rank r holds the r-th n^3 block of an n x n x (n R) mesh;
    --strong: the n^3 mesh of the config split into R slabs."""

    kernel_label = ("lattice K-M2, K-CTe, K-Q, K-Cb on the owned vertex planes + NCCL "
                    "one-plane ghost exchanges between them (lattice_slab.cu)")
    layout = "lattice"

    def __init__(self, cfg, device, rank, world, dist, strong=False, transport="nccl"):
        import paper_2301_01753_b200 as S
        from paper_2301_01753_b200 import configs, inputs
        from paper_2301_01753_b200.partition import LatticeSlab, ipc_unique_id
        t0 = time.perf_counter()
        self.scaling = "strong" if strong else "weak"
        ids = [None]
        if dist is not None and world > 1:
            new_id = ipc_unique_id if transport == "ipc" else S.nccl_unique_id
            ids = [new_id() if rank == 0 else None]
            dist.broadcast_object_list(ids, src=0)
        n = cfg["n"]
        nzg = n if strong else n * world
        self.s = LatticeSlab(n, cfg["jitter"], 2023, nzg=nzg, dt=1.0, rank=rank, nranks=world,
                             transport=transport, comm_id=ids[0], device=device)
        s = self.s
        if cfg["init"] == "gaussian":
            a = inputs.gaussian_ids(7, np.arange(s.e_glob, s.e_glob + s.n1))
        else:
            a = s.pulse(7, 0.1, cfg.get("npulses", 1))
        self.b0 = s.curl(a)
        self.e0 = np.zeros(s.n1)
        s.set_dt(configs.cfl_dt(s))
        self.dt = s.dt()
        self.n1, self.n2 = s.n1, s.n2
        self.ndof = s.n1 + s.n2  # this rank's owned DOFs
        self.setup_s = time.perf_counter() - t0
        self._stream = None

    def stream(self, torch):
        if self._stream is None:
            self._stream = torch.cuda.ExternalStream(self.s.stream_ptr())
        return self._stream

    def set_stream(self, ptr):
        pass

    def load(self):
        self.s.set_state(self.b0, self.e0)

    def advance(self, k):
        self.s.advance(k)

    def launches(self):
        return self.s.last_launches()

    def dominant(self, k_steps):
        self.s.kernel_timing(True)
        self.advance(k_steps)
        t = self.s.kernel_timing(False)
        self.per_kernel = {k: {"avg_ms": v["ms"] / max(v["launches"], 1),
                               "launches": v["launches"],
                               "bytes_per_launch": v["bytes_per_launch"],
                               "gbs": v["bytes_per_launch"] / (v["ms"] / max(v["launches"], 1)
                                                               * 1e-3) / 1e9
                               if v["ms"] > 0 else None}
                           for k, v in t.items()}
        name = max(t, key=lambda k: t[k]["ms"])
        d = t[name]
        return name, d["bytes_per_launch"], d["ms"] / max(d["launches"], 1)

    def step_bytes(self):
        return self.s.step_bytes()

    def diagnostics(self):
        return self.s.energy(), None  # collective; the whole mesh's energy

    def e2e(self, k, torch):
        t0 = time.perf_counter()
        self.s.set_state(self.b0, self.e0)
        self.advance(k)
        self.s.get_state()
        self.e2e_bytes = 8 * (self.b0.size + self.e0.size)
        return time.perf_counter() - t0


def run_ours(args, rank, world, local_rank):
    import torch

    cfg = CONFIGS[args.config]
    ipc = args.transport == "ipc"
    if ipc:  # ranks may share a GPU (host-synchronised transport)
        local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1 or args.dist:
        import torch.distributed as dist
        if ipc:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    tr = args.transport
    if cfg["kind"] == "yee":
        R = YeeRunner(cfg, local_rank, rank, world, dist, transport=tr)
    elif cfg["kind"] == "tet" and (dist is not None or args.partitioned):
        R = LatSlabRunner(cfg, local_rank, rank, world, dist, strong=args.strong, transport=tr)
    elif dist is not None or args.partitioned:
        R = TetSlabRunner(cfg, local_rank, rank, world, dist, transport=tr)  # P2-: sliced slabs
    else:
        R = TetRunner(cfg, local_rank)
    if hasattr(R, "stream"):
        stream = R.stream(torch)
    else:
        stream = torch.cuda.current_stream()
        R.set_stream(stream.cuda_stream)
    rdev = "cpu" if ipc else "cuda"  # gloo reduces host tensors
    strong = getattr(R, "scaling", "weak") == "strong"
    if isinstance(R, LatSlabRunner):  # owned DOFs per rank: the job's total is their sum
        units = R.ndof
        if dist:
            t_ = torch.tensor([float(R.ndof)], device=rdev, dtype=torch.float64)
            dist.all_reduce(t_)
            units = int(t_.item())
    else:
        units = R.ndof if strong else world * R.ndof  # DOFs the whole job advances per step
    R.load()
    energy0, gauss0 = R.diagnostics()
    R.advance(args.warmup)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        start.record(stream)
        R.advance(args.steps)
        end.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = start.elapsed_time(end)
    launches = R.launches()
    energy1, gauss1 = R.diagnostics()  # untimed: the state after warmup + steps
    if dist and not isinstance(R, LatSlabRunner):  # (the lattice slabs' energy is collective)
        t = torch.tensor([energy0, energy1], device=rdev, dtype=torch.float64)
        dist.all_reduce(t)  # each rank holds its part of the energy sums
        energy0, energy1 = float(t[0]), float(t[1])
    # dominant kernel: average launch duration with CUDA events on the launch stream
    kname, kbytes, k_avg_ms = R.dominant(min(args.steps, 200))
    if dist:
        t = torch.tensor([ms, k_avg_ms], device=rdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, k_avg_ms = float(t[0]), float(t[1])
    if dist:
        dist.barrier()
    R.e2e(max(1, min(args.warmup, args.steps)), torch)  # untimed: first-call costs
    if dist:
        dist.barrier()
    e2e_s = R.e2e(args.steps, torch)
    if dist:
        t = torch.tensor([e2e_s], device=rdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])

    trname = ("CUDA-IPC (host-synchronised; ranks share GPUs: functional check)" if ipc
              else "NCCL")
    peak, peak_src = hbm_peak()
    # roofline of the dominant kernel: DRAM bytes per launch (ncu, committed
    # under profiles/) over the CUDA-event launch time; the algorithmic count
    # (SURVEY.md 8(d) bytes per launch) over the same time beside it
    alg_achieved = kbytes / (k_avg_ms * 1e-3) / 1e9
    traffic = committed_traffic(args.config, getattr(R, "layout", None))
    achieved = traffic / (k_avg_ms * 1e-3) / 1e9 if traffic else alg_achieved
    ndof = R.ndof
    value = units * args.steps / (ms * 1e-3)
    step_gbs = R.step_bytes() / (ms / args.steps * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": cfg["dtype"],
        "data": "synthetic (seeded: " + ("Gaussian A" if cfg.get("init", "gaussian") ==
                                         "gaussian" else "Gaussian pulse A")
                + ", B0 = C A, E0 = 0)",
        "config": {"workload": f"{args.config}: {cfg['desc']}" + (
                       f" per GPU (global {cfg['n']}x{cfg['n']}x{cfg['n'] * world})"
                       if world > 1 and not strong else (" (whole mesh over all GPUs)"
                                                         if world > 1 else "")),
                   "dofs_per_gpu": ndof if not strong else ndof / world,
                   "n1_edges": R.n1, "n2_faces": R.n2, "dt": R.dt,
                   "parallelism": (f"z-slabs x{world}, {trname} ghost exchange" if cfg["kind"] == "yee"
                                   else f"z-slabs x{world} of the Kuhn lattice, per-rank "
                                        f"assembly, {trname} one-plane ghost exchanges"
                                   if isinstance(R, LatSlabRunner)
                                   else f"z-slabs x{world}, {trname} halo-plane exchange")
                                  if world > 1 else "single GPU",
                   "l2": "inputs larger than L2" if R.step_bytes() > 126e6 * 2
                         else "working set fits in L2 (latency-bound parity config)",
                   "kernel": R.kernel_label},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "basis": ("ncu dram__bytes_read+write per launch (profiles/traffic.json) / "
                               "CUDA-event average launch time" if traffic else
                               "algorithmic bytes per launch / CUDA-event average launch time"),
                     "algorithmic_achieved": alg_achieved, "algorithmic_frac": alg_achieved / peak,
                     "kernel": kname, "bytes_per_launch": kbytes, "kernel_avg_ms": k_avg_ms,
                     "step_bytes": R.step_bytes(), "step_achieved_gbs": step_gbs,
                     "peak_source": peak_src},
        "e2e": {"value": units * args.steps / e2e_s, "unit": UNIT,
                # the state crosses PCIe once per job (set_state ... get_state);
                # per step that is the job's bytes / steps
                "h2d_bytes_per_step": int(getattr(R, "e2e_bytes", 8 * ndof)) // args.steps,
                "d2h_bytes_per_step": int(getattr(R, "e2e_bytes", 8 * ndof)) // args.steps,
                "h2d_bytes_per_job": int(getattr(R, "e2e_bytes", 8 * ndof)),
                "d2h_bytes_per_job": int(getattr(R, "e2e_bytes", 8 * ndof)),
                "job": f"set_state (pinned host -> HBM) + advance({args.steps}) + get_state "
                       "(HBM -> pinned host) through the C ABI, one job timed by wall clock"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        # discrete energy 1/2 (eps0 e.Q e + b.M2 b / mu0) before the first and
        # after the last step (warmup + timed), device-side, outside the timed
        # region; leapfrog keeps it bounded (a modified energy is conserved)
        "physics": {"energy_0": energy0, "energy_end": energy1,
                    "steps": args.warmup + args.steps,
                    "rel_energy_change": (energy1 - energy0) / energy0 if energy0 else None,
                    "gauss_residual_0": gauss0, "gauss_residual_end": gauss1,
                    "gauss_rel": (gauss1 / float(np.abs(R.b0).max())
                                  if gauss1 is not None and R.b0.size else None),
                    "note": "bounded oscillation, not drift: the leapfrog conserves a modified "
                            "energy; white-noise A (Gaussian init) puts energy at the grid "
                            "Nyquist frequency where the two differ most, a smooth pulse does "
                            "not"},
    }
    if hasattr(R, "per_kernel"):
        line["roofline"]["per_kernel"] = R.per_kernel
    if hasattr(R, "setup_s"):
        line["config"]["host_setup_s"] = R.setup_s
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference_sample(args.config, budget_s=args.cpu_budget)
    if rank == 0:
        emit(line)
    if dist:
        dist.destroy_process_group()


def committed_traffic(config, layout=None):
    """ncu dram bytes per launch of the dominant kernel, from profiles/ (or None);
    keyed config/layout for the tet configs (lattice or sell)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{config}/{layout}" if layout else config)
    except Exception:
        return None


def _ref_operators(config):
    """(q, c, m2, b0, e0, dt, label, same_config) for the reference CPU arm,
    built WITHOUT the product library (that arm must not map it): the
    reference's own periodic cubical lattice (mesh_cubical.cpp + the Q1 curl,
    through oracle/_ref) for Yee, the C restatement oracle/tet_oracle.c for
    first-order tets, the numpy restatement oracle/p2_oracle.py for P2-."""
    from oracle import oracle as O
    cfg = CONFIGS[config]
    n = cfg["ref_n"]
    if cfg["kind"] == "yee":
        # yee_equivalence_check's lumped system (yee.cpp:95-121) on the
        # reference's periodic n^3 lattice: same per-DOF operators as the PEC
        # workload (7-point curl pairs, diagonal Q and M2), no walls
        h = 1.0 / n
        c = O.ref_cubical_curl(n, n, n, h, h, h)
        n1, n2 = c[1], c[0]
        dv = h ** 3
        q = (n1, n1, np.arange(n1 + 1), np.arange(n1, dtype=np.int32), np.full(n1, 1.0 / dv))
        m2 = (n2, n2, np.arange(n2 + 1), np.arange(n2, dtype=np.int32), np.full(n2, dv))
        a = O.port_uniform(20260101, n1)
        return (q, c, m2, O.port_spmv(c, a), np.zeros(n1), 0.5 / (np.sqrt(3.0) * n),
                f"{n}^3 periodic cubical lattice of the reference (mesh_cubical.cpp), lumped "
                "masses", n == cfg["n"])
    if cfg["kind"] == "p2":
        from oracle.p2_oracle import OracleP2
        from oracle.tetmesh_oracle import OracleTetMesh, pattern, spai_lstsq

        def csr(rows, ncols):
            rp = np.cumsum([0] + [len(r) for r in rows]).astype(np.int64)
            return (len(rows), ncols, rp, np.array([c for r in rows for c, _ in r], np.int32),
                    np.array([v for r in rows for _, v in r]))
        P = OracleP2(OracleTetMesh(n, cfg["jitter"], 2023))
        c, m1, m2 = (csr(P.curl_rows(), P.n1), csr(P.mass_rows(1), P.n1),
                     csr(P.mass_rows(2), P.n2))
        pat = pattern(m1, "m1sq")  # S(M1^2), spai.cpp:31-72
        cols = spai_lstsq(m1, pat)
        qr = np.concatenate([np.asarray(p_, np.int64) for p_ in pat])
        qc = np.repeat(np.arange(P.n1), [len(p_) for p_ in pat])
        order = np.lexsort((qc, qr))
        q = (P.n1, P.n1, np.searchsorted(qr[order], np.arange(P.n1 + 1)).astype(np.int64),
             qc[order].astype(np.int32), np.concatenate(cols)[order])
        a = O.port_uniform(7, P.n1)
        return (q, c, m2, O.port_spmv(c, a), np.zeros(P.n1), 1e-3,
                f"{n}^3 x 6 Kuhn tets (P2-, S(M1^2) SPAI; operators from the numpy "
                "restatement oracle/p2_oracle.py)", n == cfg["n"])
    r = O.tet_c_operators(n, cfg["jitter"], 2023)
    c = r["c"]
    a = O.port_uniform(7, c[1])
    return (r["q_sym"], c, r["m2"], O.port_spmv(c, a), np.zeros(c[1]), 1e-3,
            f"{n}^3 x 6 Kuhn tets (P1-, S(M1) SPAI; operators from the C restatement "
            "oracle/tet_oracle.c)", n == cfg["n"])


def _omp_threads(k):
    """Set the OpenMP thread count of this process (libgomp, shared by the
    reference library)."""
    import ctypes as C
    C.CDLL("libgomp.so.1").omp_set_num_threads(int(k))


def cpu_reference_sample(config, budget_s=20.0, max_steps=1000, threads=None):
    """The reference SplitScheme::step (oracle/_ref, unmodified reference
    sources) on the same per-DOF workload, timed on the host cores: with all
    host threads (`value`) and with one (`value_1thread`)."""
    from oracle import oracle as O
    cores = os.cpu_count()
    if not O.ref_available():
        return {"value": None, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": "oracle/_ref missing"}
    t0 = time.perf_counter()
    q, c, m2, b, e, dt, label, same = _ref_operators(config)
    ref = O.RefScheme(1, dt, q, c, m2)
    setup_s = time.perf_counter() - t0
    n1, n2 = c[1], c[0]

    def timed(nthreads, budget):
        nonlocal b, e
        _omp_threads(nthreads)
        b, e, _, _ = ref.steps(True, b, e, 1)  # warm-up
        steps, secs = 0, 0.0
        while secs < budget and steps < max_steps:
            b, e, _, _ = ref.steps(True, b, e, 1)
            secs += ref.last_seconds
            steps += 1
        return (n1 + n2) * steps / secs, steps, secs

    v_all, k_all, s_all = timed(threads or cores, budget_s)
    v_one, k_one, s_one = timed(1, max(budget_s / 2, 5.0))
    _omp_threads(cores)
    return {"value": v_all, "unit": UNIT, "cores": threads or cores, "kind": "reference",
            "value_1thread": v_one,
            "same_config": bool(same),
            "sample": f"{k_all} x reference SplitScheme::step (Strang, BE) on the {label} "
                      f"(N1+N2={n1 + n2}), wall clock {s_all:.1f} s, OpenMP threads = "
                      f"{threads or cores}; and {k_one} steps ({s_one:.1f} s) on 1 thread"
                      + ("" if same else "; the workload's own size is infeasible for the "
                         "reference (int32 triplet overflow in symmetric_part at 256^3, "
                         "BASELINE.md 5), so this is the largest feasible size, compared "
                         "per DOF") + f"; operator setup {setup_s:.0f} s untimed"}


def run_reference(args, rank, world):
    cfg = CONFIGS[args.config]
    if rank != 0:
        return
    base = cpu_reference_sample(args.config, budget_s=args.ref_budget,
                                max_steps=max(args.steps, 1))
    line = {"metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
            "data": "synthetic (seeded A, B0 = C A, E0 = 0)",
            "config": {"workload": f"{args.config}: {cfg['desc']} (reference CPU step; "
                                   "bounded per-DOF sample)"},
            "cpu_baseline": {k: base[k] for k in ("kind", "cores", "sample", "value")},
            "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if cfg.get("precision") == 4:
        line["config"]["note"] = "the reference is fp64 only"
    emit(line)


def dptr(t):
    return ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_double))


_JSON_OUT = None


def emit(line):
    """The one JSON line, on the process's original stdout."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # everything else that writes to fd 1 (NCCL's version banner, library
    # prints) goes to stderr, so stdout carries exactly the JSON line
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="tet256")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partitioned", action="store_true",
                    help="tet configs at N=1: run the z-slab partition path (one slab)")
    ap.add_argument("--strong", action="store_true",
                    help="tet configs under torchrun: split the config's mesh (strong scaling) "
                         "instead of one n^3 block per rank (weak scaling, the default)")
    ap.add_argument("--dist", action="store_true",
                    help="the multi-GPU code path (NCCL process group, slab runners, "
                         "max-over-ranks) even at world size 1, e.g. under torchrun with "
                         "one process")
    ap.add_argument("--transport", choices=["nccl", "ipc"], default="nccl",
                    help="ghost-plane transport of a multi-rank run. nccl: one GPU per rank "
                         "(the driver's launch). ipc: the product's host-synchronised CUDA-IPC "
                         "transport with gloo for the plumbing; ranks share GPUs when there "
                         "are fewer GPUs than ranks (a functional check of the multi-rank "
                         "flow on a one-GPU box, not a scaling number)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=60.0)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
