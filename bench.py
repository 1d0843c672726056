#!/usr/bin/env python
"""Benchmark of the B200 SFEEC leapfrog (BASELINE.json metric:
"edge+face DOF-updates/sec per leapfrog step; achieved HBM GB/s vs peak").

Default workload = BASELINE.json configs[1]: Yee special case, 256^3 cubical
cells, lumped masses, PEC walls, Courant 0.5, fp64; E0 = 0, B0 = C A with
seeded Gaussian A. A "step" is one leapfrog step over all N1 + N2 DOFs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config yee256|yee256_f32]

Under torchrun (N > 1) every rank runs its own 256^3 block (weak scaling).
`--impl reference` times the reference CPU step (oracle/_ref: the unmodified
reference SplitScheme::step, dynamics.cpp:69-90) on the host cores.
"""
from __future__ import annotations

import argparse
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
    "yee256": dict(n=256, precision=8, dtype="f64"),
    "yee256_f32": dict(n=256, precision=4, dtype="f32"),
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
            self._stop.wait(0.2)

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


def yee_setup(n, precision, device):
    """Operators + initial state of configs[1] on an n^3 unit cube."""
    import paper_2301_01753_b200 as S
    from paper_2301_01753_b200 import inputs
    h = 1.0 / n
    dt = 0.5 / (np.sqrt(3.0) * n)  # Courant 0.5: c dt sqrt(sum 1/d^2) = 0.5
    y = S.YeeScheme(n, n, n, h, h, h, dt, bc=1, precision=precision, device=device)
    a = inputs.gaussian(20260101, y.n_edges)
    # B0 = C A, computed on the device: a b-kick with h = -dV from e = A gives
    # b = -h * C Q A = C A (Q = I/dV)
    y.load(np.zeros(y.n_faces), a)
    y.flow_he(-(h ** 3))
    b0, _, _ = y.fetch()
    e0 = np.zeros(y.n_edges)
    return y, b0, e0, dt


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2301_01753_b200 as S
    from paper_2301_01753_b200 import _lib as L

    cfg = CONFIGS[args.config]
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    y, b0, e0, dt = yee_setup(cfg["n"], cfg["precision"], local_rank)
    stream = torch.cuda.current_stream()
    L.check(L.lib().sfeec_yee_set_stream(y.handle, C_void(stream.cuda_stream)))
    y.load(b0, e0)
    ndof = y.n_edges + y.n_faces
    step_bytes = y.step_bytes()

    y.advance(args.warmup)
    torch.cuda.synchronize()
    L.check(L.lib().sfeec_yee_kernel_timing(y.handle, 1, None, None))
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        start.record(stream)
        y.advance(args.steps)
        end.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = start.elapsed_time(end)
    launches = y.last_launches()
    kms, kl = ctypes_double(), ctypes_int64()
    L.check(L.lib().sfeec_yee_kernel_timing(y.handle, 0, kms, kl))
    k_avg_ms = kms.value / max(kl.value, 1)
    if dist:
        t = torch.tensor([ms, k_avg_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, k_avg_ms = float(t[0]), float(t[1])

    # end to end through the C ABI: pinned host state -> device, K steps, -> host
    pin_b = torch.from_numpy(b0).pin_memory()
    pin_e = torch.from_numpy(e0).pin_memory()
    out_b = torch.empty_like(pin_b).pin_memory()
    out_e = torch.empty_like(pin_e).pin_memory()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    L.check(L.lib().sfeec_yee_set_state(y.handle, dptr(pin_b), dptr(pin_e), 0.0))
    y.advance(args.steps)
    L.check(L.lib().sfeec_yee_get_state(y.handle, dptr(out_b), dptr(out_e), None))
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])

    peak, peak_src = hbm_peak()
    achieved = step_bytes / (k_avg_ms * 1e-3) / 1e9
    value = world * ndof * args.steps / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": cfg["dtype"], "data": "synthetic (seeded Gaussian A, B0 = C A, E0 = 0)",
        "config": {"workload": f"{args.config}: BASELINE configs[1] Yee/lumped-mass SFEEC, "
                               f"{cfg['n']}^3 cells per GPU, PEC, Courant 0.5",
                   "dofs_per_gpu": ndof, "n1_edges": y.n_edges, "n2_faces": y.n_faces,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (fields %.0f MB per buffer)"
                         % (ndof * cfg["precision"] / 1e6),
                   "kernel": "fused e-kick + b-kick z-sweep (k_fused_pec)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": committed_traffic(args.config),
                     "bytes_per_step": step_bytes, "kernel_avg_ms": k_avg_ms,
                     "peak_source": peak_src},
        "e2e": {"value": world * ndof * args.steps / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(8 * ndof), "d2h_bytes_per_step": int(8 * ndof),
                "job": f"set_state + advance({args.steps}) + get_state via the C ABI, "
                       "pinned host buffers"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference_sample(budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def committed_traffic(config):
    """ncu dram bytes per launch of the dominant kernel, from profiles/ (or None)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(config)
    except Exception:
        return None


def cpu_reference_sample(budget_s=20.0, n=128, max_steps=1000):
    """The reference SplitScheme::step (oracle/_ref, unmodified reference
    sources) on the same per-DOF workload, timed on the host cores."""
    from oracle import oracle as O
    import paper_2301_01753_b200 as S
    if not O.ref_available():
        return {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                "sample": "oracle/_ref missing"}
    h = 1.0 / n
    c, _ = S.yee_operators(n, n, n, h, h, h, bc=1)
    dv = h ** 3
    n1, n2 = c.cols, c.rows
    q = (n1, n1, np.arange(n1 + 1), np.arange(n1, dtype=np.int32), np.full(n1, 1.0 / dv))
    m2 = (n2, n2, np.arange(n2 + 1), np.arange(n2, dtype=np.int32), np.full(n2, dv))
    dt = 0.5 / (np.sqrt(3.0) * n)
    ref = O.RefScheme(1, dt, q, (c.rows, c.cols, c.row_ptr, c.col_idx, c.val), m2)
    from paper_2301_01753_b200 import inputs
    a = inputs.gaussian(20260101, n1)
    b = O.ref_spmv((c.rows, c.cols, c.row_ptr, c.col_idx, c.val), a)
    e = np.zeros(n1)
    b, e, _, _ = ref.steps(True, b, e, 1)  # warm-up
    steps, secs = 0, 0.0
    while secs < budget_s and steps < max_steps:
        b, e, _, _ = ref.steps(True, b, e, 1)
        secs += ref.last_seconds
        steps += 1
    return {"value": (n1 + n2) * steps / secs, "unit": UNIT, "cores": os.cpu_count(),
            "kind": "reference",
            "sample": f"{steps} x reference SplitScheme::step (Strang, BE) on the {n}^3 PEC "
                      f"lattice (N1+N2={n1 + n2}), wall clock, OpenMP threads = all "
                      f"{os.cpu_count()} host cores; same per-DOF operators as 256^3"}


def run_reference(args, rank, world):
    cfg = CONFIGS[args.config]
    if rank != 0:
        return
    base = cpu_reference_sample(budget_s=args.ref_budget)
    line = {"metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
            "data": "synthetic (seeded Gaussian A, B0 = C A, E0 = 0)",
            "config": {"workload": f"{args.config}: BASELINE configs[1] Yee/lumped-mass SFEEC "
                                   "(reference CPU step; bounded per-DOF sample)"},
            "cpu_baseline": {k: base[k] for k in ("kind", "cores", "sample", "value")},
            "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if cfg["precision"] == 4:
        line["config"]["note"] = "the reference is fp64 only"
    print(json.dumps(line), flush=True)


# small ctypes helpers
def C_void(p):
    import ctypes
    return ctypes.c_void_p(p)


def ctypes_double():
    import ctypes
    return ctypes.c_double()


def ctypes_int64():
    import ctypes
    return ctypes.c_int64()


def dptr(t):
    import ctypes
    return ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_double))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="yee256")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
