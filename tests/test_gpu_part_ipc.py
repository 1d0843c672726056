"""GPU: the sliced z-slab leapfrog (csrc/partition.cu: the multi-rank path of
config 4, P2- with a two-plane halo, and of the sliced first-order kernels)
across real PROCESSES through the product's own exchange code. R = 2 and 3
processes, all on cuda:0, each a TetPart assembled and row-sliced on the
device, with the CUDA-IPC transport (sfeec_part_attach_ipc: the neighbours'
e, t, b, u mapped, halo rows pulled between host-side barriers), advance
bitwise equal to the single-GPU device scheme (P2- at n = 5, first order at
n = 9; 1e-13 where a slab's operator parts pick another SpMV layout)."""
import multiprocessing as mp

import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200 import configs, inputs
from paper_2301_01753_b200.partition import ipc_unique_id

pytestmark = pytest.mark.gpu


def _run(nranks, cfg):
    if cfg["order"] == 2:
        one = S.p2_device_scheme(cfg["n"], cfg["jitter"], cfg["seed"], dt=1.0, with_div=False,
                                 layout="sell")
    else:
        one = S.tet_device_scheme(cfg["n"], cfg["jitter"], seed=cfg["seed"], dt=1.0,
                                  with_div=False, layout="sell")
    dt = configs.cfl_dt(one)
    one.set_dt(dt)
    b0 = one.apply("c", inputs.gaussian(7, one._n1))
    e0 = np.random.default_rng(1).standard_normal(one._n1)
    ref = one.advance(S.make_state(S.Formulation.BE, b0, e0), cfg["steps"])
    ren = one.energy(ref)
    del one
    from tests.part_worker import run_rank
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    cid = ipc_unique_id()
    procs = [ctx.Process(target=run_rank, args=(r, nranks, cid, cfg, b0, e0, q))
             for r in range(nranks)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(nranks):
            item = q.get(timeout=900)
            res[item[0]] = item
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    errs = [r[-1] for r in res.values() if r[-1]]
    assert not errs, errs
    b, e = np.full(b0.size, np.nan), np.full(e0.size, np.nan)
    en = 0.0
    for r in range(nranks):
        _, eg, fg, bb, ee, t, en_r, dt_r, _ = res[r]
        b[fg[1]:fg[2]] = bb
        e[eg[1]:eg[2]] = ee
        en += en_r
        assert dt_r == dt and t == ref.time
    if cfg.get("tol") is None:
        assert np.array_equal(b, ref.first) and np.array_equal(e, ref.e)
    else:  # (larger P2 slabs pick other SpMV layouts than the whole operator: last-bit sums)
        assert np.abs(b - ref.first).max() <= cfg["tol"] * np.abs(ref.first).max()
        assert np.abs(e - ref.e).max() <= cfg["tol"] * np.abs(ref.e).max()
    assert en == pytest.approx(ren, rel=1e-12)


@pytest.mark.parametrize("nranks", [2, 3])
def test_p2_slab_processes_equal_single_device(nranks):
    """config 4's path: two-plane halo, S(M1^2) Q"""
    _run(nranks, dict(n=5, jitter=0.1, seed=2023, order=2, steps=11))


def test_p2_slab_processes_larger_mesh():
    """n = 7: each slab's operator parts choose their own sliced / ELL layout,
    so rows may sum in another order than the whole operator's: 1e-13, as the
    lockstep slabs on one device give"""
    _run(2, dict(n=7, jitter=0.1, seed=2023, order=2, steps=11, tol=1e-13))


@pytest.mark.parametrize("nranks", [2, 3])
def test_tet_sliced_slab_processes_equal_single_device(nranks):
    _run(nranks, dict(n=9, jitter=0.1, seed=5, order=1, steps=14))
