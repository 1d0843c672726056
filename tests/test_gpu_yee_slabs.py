"""GPU: the z-slab Yee / FDTD leapfrog (config 2's multi-GPU path, yee.cu;
SURVEY.md 8(e)) across real PROCESSES through the product's own exchange code.
R = 2 and 3 processes, all on cuda:0, each a YeeSlab with the CUDA-IPC
transport (the neighbours' ping-pong buffers mapped, ghost planes pulled
between host-side barriers; no kernel waits on another rank), advance bitwise
equal to the single-domain scheme, for the one-step sweeps (variants 0, 2) and
the default two-step TMA sweep (variant 4), fp64 and fp32. The NCCL transport
moves the same planes (exchange_nccl); it needs one GPU per rank."""
import multiprocessing as mp

import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200.partition import ipc_unique_id

pytestmark = pytest.mark.gpu


def _run(nranks, cfg):
    dims = cfg["dims"]
    c, _ = S.yee_operators(*dims, *cfg["h"], bc=1)
    rng = np.random.default_rng(cfg.get("seed", 3))
    from paper_2301_01753_b200.configs import spmv
    b0 = spmv(c, rng.standard_normal(c.cols))  # B0 = C A: discretely divergence-free
    e0 = rng.standard_normal(c.cols)
    from tests.envutil import layout_env
    env = {} if cfg.get("variant") is None else {"SFEEC_YEE_VARIANT": cfg["variant"]}
    with layout_env(**env):
        ref = S.YeeScheme(*dims, *cfg["h"], cfg["dt"], bc=1, precision=cfg["precision"])
        ref.load(b0, e0)
        ref.advance(cfg["steps"])
        rb, re_, rt = ref.fetch()
        ren = ref.energy()
        del ref
    from tests.yee_slab_worker import run_rank
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
            item = q.get(timeout=600)
            res[item[0]] = item
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    errs = [r[-1] for r in res.values() if r[-1]]
    assert not errs, errs
    b, e = np.full_like(rb, np.nan), np.full_like(re_, np.nan)
    en = 0.0
    for r in range(nranks):
        _, em, fm, bb, ee, t, en_r, _ = res[r]
        b[fm] = bb
        e[em] = ee
        en += en_r
        assert t == rt
    assert np.array_equal(b, rb) and np.array_equal(e, re_)  # bitwise the single domain
    assert en == pytest.approx(ren, rel=1e-12)  # (each rank sums its own planes)


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("variant", [4, 2, 0])
def test_yee_slab_processes_equal_single_domain(nranks, variant):
    _run(nranks, dict(dims=(40, 36, 12 * nranks), h=(1.0, 0.8, 1.25), dt=0.2, steps=9,
                      precision=8, variant=variant))


def test_yee_slab_processes_default_variant_even_steps_fp32():
    _run(2, dict(dims=(64, 33, 16), h=(0.5, 0.5, 0.5), dt=0.1, steps=12, precision=4,
                 variant=None))
