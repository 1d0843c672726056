"""GPU: the multi-rank lattice leapfrog (csrc/lattice_slab.cu; SURVEY.md
8(e)). Each rank assembles only its own z-slab of the mesh; ranks exchange
one-plane ghosts after each kernel and combine plane sums in plane order.

* one rank of the slab code equals the single-GPU lattice handle bitwise;
* R = 2 and 3 PROCESSES (one GPU; the product's CUDA-IPC transport, host-
  synchronised -- no kernel waits on another rank) advance bitwise equal to
  one rank: the same states, energy and CFL number, on the unit cube (strong
  split) and on a weak-scaling stack n x n x (n R).
"""
import multiprocessing as mp

import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200.partition import LatticeSlab, ipc_unique_id

pytestmark = pytest.mark.gpu


def _state(n1, n2, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(n2), rng.standard_normal(n1)


def test_one_rank_slab_equals_single_gpu_lattice():
    n, dt = 12, 0.01
    one = LatticeSlab(n, 0.1, 3, dt=dt)
    ref = S.tet_device_scheme(n, 0.1, 3, dt=dt, layout="lattice")
    assert (one.n1, one.n2) == (ref._n1, ref._n2) and one.e_glob == one.f_glob == 0
    b0, e0 = _state(one.n1, one.n2, 1)
    one.set_state(b0, e0)
    one.advance(23)
    b, e, t = one.get_state()
    out = ref.advance(S.make_state(S.Formulation.BE, b0, e0), 23)
    assert np.array_equal(b, out.first) and np.array_equal(e, out.e)
    assert t == out.time
    assert one.energy() == pytest.approx(ref.energy(out), rel=1e-13)
    assert one.cfl_number() == pytest.approx(ref.cfl_number(), rel=1e-12)
    # B0 = C A through the slab equals the handle's C
    a = np.random.default_rng(5).standard_normal(one.n1)
    assert np.array_equal(one.curl(a), ref.apply("c", a))


def _multi(nranks, cfg):
    ref = LatticeSlab(cfg["n"], cfg["jitter"], cfg["seed"], nzg=cfg["nzg"], dt=cfg["dt"],
                      kind=cfg["kind"])
    b0, e0 = _state(ref.n1, ref.n2, 7)
    ref.set_state(b0, e0)
    cfl = ref.cfl_number()
    ref.advance(cfg["steps"])
    en = ref.energy()
    rb, re_, rt = ref.get_state()
    del ref
    from tests.slab_worker import run_rank
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
    b = np.zeros_like(rb)
    e = np.zeros_like(re_)
    for r in range(nranks):
        _, eg, fg, bb, ee, t, en_r, cfl_r, assembled, planes, _ = res[r]
        b[fg:fg + bb.size] = bb
        e[eg:eg + ee.size] = ee
        assert t == rt and en_r == en and cfl_r == cfl  # bitwise, every rank
        # the rank assembled only its slab (4 planes beyond its owned ones)
        assert assembled[0] >= planes[0] - 4 and assembled[1] <= planes[1] + 4
    assert np.array_equal(b, rb) and np.array_equal(e, re_)


@pytest.mark.parametrize("nranks", [2, 3])
def test_processes_over_ipc_equal_one_rank_unit_cube(nranks):
    _multi(nranks, dict(n=10, nzg=10, jitter=0.12, seed=11, dt=0.01, kind=1, steps=17))


def test_processes_over_ipc_equal_one_rank_weak_stack():
    """config 5's weak-scaling mesh shape: n x n x (n R), one n^3 block per rank"""
    _multi(2, dict(n=8, nzg=16, jitter=0.1, seed=4, dt=0.01, kind=1, steps=12))


def test_processes_lie_trotter():
    _multi(2, dict(n=7, nzg=7, jitter=0.1, seed=2, dt=0.02, kind=0, steps=9))


def test_processes_serialised_exchange():
    """SFEEC_PART_OVERLAP=0: the exchange after the whole kernel instead of
    beside its interior planes -- the same bitwise result"""
    from tests.envutil import layout_env
    with layout_env(SFEEC_PART_OVERLAP=0):
        _multi(2, dict(n=9, nzg=9, jitter=0.1, seed=8, dt=0.01, kind=1, steps=10))
