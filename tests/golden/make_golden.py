"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run here (the reference is only present in the build container):
    python tests/golden/make_golden.py
Outputs tests/golden/*.npz. Inputs are seeded (splitmix64 Rng of
core.hpp:44-63 for fields, numpy default_rng for synthetic operator values);
every output array is produced by the reference's own code:
  cubical_curl.npz   generate_cubical_lattice + Q1 entry rule (mesh_cubical.cpp,
                     operators.cpp:37) on three lattices
  scheme.npz         SplitScheme (dynamics.cpp) on synthetic operators built on
                     the reference periodic lattice: 4 (kind, formulation)
                     cases x (state after 20 steps, energy history, CFL,
                     Q_sym, one flow_he / flow_ha)
  yee.npz            YeeGrid FDTD (yee.cpp) 3x4x5, 60 steps, and the lumped
                     SplitScheme on the same data (yee_equivalence_check's recipe)
  triplets.npz       operator_from_triplets with duplicates / cancellations
"""
from __future__ import annotations

import os
import sys

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def to_sp(a):
    rows, cols, rp, ci, va = a
    return sp.csr_matrix((va, ci, rp), shape=(rows, cols))


def from_sp(m):
    m = sp.csr_matrix(m)
    m.sort_indices()
    return (m.shape[0], m.shape[1], m.indptr.astype(np.int64), m.indices.astype(np.int32),
            m.data.astype(np.float64))


def synthetic_ops(n=3, seed=0):
    """C from the reference periodic lattice; M2 SPD on the C C^T pattern; Q
    nonsymmetric on the C^T C pattern (so symmetric_part is exercised)."""
    rng = np.random.default_rng(seed)
    c = O.ref_cubical_curl(n, n, n, 1.0, 1.0, 1.0)
    cs = to_sp(c)
    pat2 = (abs(cs) @ abs(cs).T).tocsr()
    pat2.data[:] = 1.0
    r = sp.triu(pat2, 1).tocoo()
    vals = rng.uniform(-0.1, 0.1, r.nnz)
    off = sp.coo_matrix((vals, (r.row, r.col)), shape=pat2.shape)
    m2 = (off + off.T + sp.identity(pat2.shape[0]) * 2.0).tocsr()
    pat1 = (abs(cs).T @ abs(cs)).tocsr().tocoo()
    qv = rng.uniform(-0.05, 0.05, pat1.nnz)
    q = sp.coo_matrix((qv, (pat1.row, pat1.col)), shape=pat1.shape).tocsr()
    q = q + sp.identity(q.shape[0]) * 1.0
    return from_sp(q), c, from_sp(m2), cs


def main():
    out = {}
    for tag, (nx, ny, nz, dx, dy, dz) in {
        "unit4": (4, 4, 4, 1.0, 1.0, 1.0),
        "aniso345": (3, 4, 5, 1.0, 0.5, 2.0),
        "nondyadic": (3, 2, 4, 0.1, 0.3, 0.7),
    }.items():
        rows, cols, rp, ci, va = O.ref_cubical_curl(nx, ny, nz, dx, dy, dz)
        out[f"{tag}_dims"] = np.array([nx, ny, nz])
        out[f"{tag}_d"] = np.array([dx, dy, dz])
        out[f"{tag}_rp"], out[f"{tag}_ci"], out[f"{tag}_va"] = rp, ci, va
    np.savez_compressed(os.path.join(OUT, "cubical_curl.npz"), **out)

    # SplitScheme cases
    q, c, m2, cs = synthetic_ops()
    n1, n2 = c[1], c[0]
    out = {"q_rp": q[2], "q_ci": q[3], "q_va": q[4], "c_rp": c[2], "c_ci": c[3], "c_va": c[4],
           "m2_rp": m2[2], "m2_ci": m2[3], "m2_va": m2[4], "n1": n1, "n2": n2}
    a0 = O.port_uniform(11, n1)
    e0 = O.port_uniform(12, n1)
    b0 = cs @ a0
    out["a0"], out["e0"], out["b0"] = a0, e0, b0
    dt, steps = 0.05, 20
    for strang in (1, 0):
        for be in (1, 0):
            s = O.RefScheme(strang, dt, q, c, m2)
            first = b0 if be else a0
            f1, e1, t1, hist = s.steps(be, first, e0, steps, energy=True)
            key = f"s{strang}b{be}"
            out[f"{key}_first"], out[f"{key}_e"], out[f"{key}_t"] = f1, e1, t1
            out[f"{key}_energy"] = hist
            out[f"{key}_energy0"] = s.energy(be, first, e0)
            fh, eh = s.flow(0, be, first, e0, 0.34)
            out[f"{key}_flowhe_first"], out[f"{key}_flowhe_e"] = fh, eh
            fa, ea = s.flow(1, be, first, e0, 0.7)
            out[f"{key}_flowha_first"], out[f"{key}_flowha_e"] = fa, ea
            out[f"{key}_cfl"] = s.cfl()
    qs = O.RefScheme(1, dt, q, c, m2).q_sym()
    out["qsym_rp"], out["qsym_ci"], out["qsym_va"] = qs[2], qs[3], qs[4]
    np.savez_compressed(os.path.join(OUT, "scheme.npz"), **out)

    # Yee FDTD and lumped SplitScheme, yee_equivalence_check recipe (yee.cpp:83-135)
    nx, ny, nz, d, dt, steps, seed = 3, 4, 5, (1.0, 0.5, 2.0), 0.15, 60, 7
    nc = nx * ny * nz
    u = O.port_uniform(seed, 6 * nc)
    e0, bgrid0 = u[:3 * nc], u[3 * nc:]
    dv = d[0] * d[1] * d[2]
    g = O.RefYee(nx, ny, nz, *d)
    g.set(e0, bgrid0)
    g.advance_b(0.5 * dt)
    g.step(dt, steps)
    e_fdtd, b_fdtd = g.get()
    c = O.ref_cubical_curl(nx, ny, nz, *d)
    n = 3 * nc
    qd = (n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.full(n, 1.0 / dv))
    md = (n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.full(n, dv))
    s = O.RefScheme(1, dt, qd, c, md)
    b0 = bgrid0 / dv
    bs, es, ts, hist = s.steps(1, b0, e0, steps, energy=True)
    bh, _ = s.flow(0, 1, bs, es, 0.5 * dt)
    np.savez_compressed(os.path.join(OUT, "yee.npz"), dims=np.array([nx, ny, nz]),
                        d=np.array(d), dt=dt, steps=steps, seed=seed, e0=e0, bgrid0=bgrid0,
                        e_fdtd=e_fdtd, b_fdtd=b_fdtd, e_sfeec=es, b_sfeec=bs,
                        b_sfeec_staggered=bh, energy=hist, t=ts)

    # operator_from_triplets with duplicates, cancellations and unsorted input
    rng = np.random.default_rng(3)
    r = rng.integers(0, 7, 60)
    cc = rng.integers(0, 5, 60)
    v = rng.choice([-1.5, -0.5, 0.5, 1.5, 0.1, 0.2], 60)
    r = np.concatenate([r, [2, 2]])
    cc = np.concatenate([cc, [3, 3]])
    v = np.concatenate([v, [1.0, -1.0]])
    m = O.ref_from_triplets(7, 5, r, cc, v)
    np.savez_compressed(os.path.join(OUT, "triplets.npz"), r=r, c=cc, v=v, rp=m[2], ci=m[3],
                        va=m[4])
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
