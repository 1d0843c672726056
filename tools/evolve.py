#!/usr/bin/env python
"""GPU counterpart of the reference's `sfeec evolve` (tools/sfeec_main.cpp:151-216):
advance a configuration and write `step,time,energy,gauss_residual` every
--diag-every steps with %.17g (sfeec_main.cpp:193-215), all on the device
(SplitScheme::advance_diag -> energy and D b reductions on the B200).

  python tools/evolve.py --config tet16 --steps 100 --diag-every 10 --out evolve.csv
  python tools/evolve.py --config yee --n 64 --steps 1000 --diag-every 100

Configs: tetN (N^3 x 6 Kuhn tets, S(M1) SPAI, device-assembled; dt = 0.5 CFL
unless --dt) and yee (PEC Yee lattice, Courant 0.5, --n cells per axis).
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tet16")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--jitter", type=float, default=0.1)
    ap.add_argument("--seed", type=int, default=2023)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--diag-every", type=int, default=10)
    ap.add_argument("--dt", type=float, default=None)
    ap.add_argument("--init", choices=["gaussian", "pulse"], default="gaussian")
    ap.add_argument("--out", default="-")
    args = ap.parse_args()

    import paper_2301_01753_b200 as S
    from paper_2301_01753_b200 import configs, inputs

    rows = []
    if args.config.startswith("tet"):
        n = args.n or int(args.config[3:] or 16)
        s = S.tet_device_scheme(n, args.jitter, args.seed, dt=1.0, with_div=True)
        mesh = S.TetMesh(n, args.jitter, args.seed)
        xyz, ev, _, _ = mesh.geometry(faces=False, tets=False)
        a = (inputs.gaussian(7, s._n1) if args.init == "gaussian"
             else inputs.pulse_one_form(xyz, ev, 7))
        b0 = s.apply("c", a)
        s.set_dt(args.dt if args.dt else configs.cfl_dt(s))
        state = S.make_state(S.Formulation.BE, b0, np.zeros(s._n1))
        # the package driver: time accumulated per step on the device (as
        # cmd_evolve's time += dt) and a final row at step == steps
        from paper_2301_01753_b200.evolve import evolve
        text = evolve(s, state, args.steps, args.diag_every)
        fh = sys.stdout if args.out == "-" else open(args.out, "w")
        fh.write(text)
        if fh is not sys.stdout:
            fh.close()
        return
    elif args.config == "yee":
        import bench
        n = args.n or 64
        y, b0, e0, dt = bench.yee_setup(n, 8, 0)
        h = 1.0 / n
        _, d = S.yee_operators(n, n, n, h, h, h)
        y.load(b0, e0)

        def gauss(b):
            rr = np.repeat(np.arange(d.rows), np.diff(d.row_ptr))
            db = np.zeros(d.rows)
            np.add.at(db, rr, d.val * b[d.col_idx])
            return np.abs(db).max()

        rows.append((0, 0.0, y.energy(), gauss(b0)))
        s = 0
        while s < args.steps:  # every diag_every steps and at the last step
            nxt = min(args.steps, (s // args.diag_every + 1) * args.diag_every)
            y.advance(nxt - s)
            s = nxt
            b, _, t = y.fetch()
            rows.append((s, t, y.energy(), gauss(b)))
    else:
        raise SystemExit(f"unknown config {args.config}")

    fh = sys.stdout if args.out == "-" else open(args.out, "w")
    fh.write("step,time,energy,gauss_residual\n")
    for step, t, e, g in rows:
        fh.write(f"{step},{t:.17g},{e:.17g},{g:.17g}\n")
    if fh is not sys.stdout:
        fh.close()


if __name__ == "__main__":
    main()
