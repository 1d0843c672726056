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
@pytest.mark.parametrize("variant", [2, 0, 4])
@pytest.mark.parametrize("steps", [30, 31])
def test_group_lockstep_bitwise_equals_single_domain(world, variant, steps):
    """Slabs with two ghost planes, the NCCL path's split schedule (boundary
    chunks, exchange, interior chunks); variant 4 = two steps per sweep."""
    dims, d = (37, 21, 70 * world), (1.0, 0.9, 1.1)  # 3 z-chunks per slab: boundary + interior
    rng = np.random.default_rng(world)
    one = S.YeeScheme(*dims, *d, 0.2, bc=1)
    one.set_variant(variant)
    b0, e0 = rng.standard_normal(one.n_faces), rng.standard_normal(one.n_edges)
    one.load(b0, e0)
    one.advance(steps)
    b1, e1, _ = one.fetch()
    grp = S.YeeGroup(*dims, *d, 0.2, world)
    grp.set_variant(variant)
    grp.load(b0, e0)
    grp.advance(steps)
    b2, e2 = grp.fetch()
    assert np.array_equal(b1, b2) and np.array_equal(e1, e2)
    assert grp.energy() == pytest.approx(one.energy(), rel=1e-13)


# ---------------------------------------------------------------------------
# tet mesh: z-slab partition with one-plane halos
# ---------------------------------------------------------------------------
from paper_2301_01753_b200 import configs, partition  # noqa: E402


def _csr(a):
    import scipy.sparse as sp
    return sp.csr_matrix((a.val, a.col_idx, a.row_ptr), shape=(a.rows, a.cols))


@pytest.fixture(scope="module")
def tet_sys():
    return configs.tet_system(7, 0.1, seed=11)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_tet_slab_operators_reproduce_global_rows(tet_sys, world):
    qs = S.symmetric_part(tet_sys.q)
    ct = S.transpose(tet_sys.c)
    rng = np.random.default_rng(0)
    xe, xf = rng.standard_normal(tet_sys.n1), rng.standard_normal(tet_sys.n2)
    owned_e, owned_f = [], []
    for r in range(world):
        ls = partition.slab_system(tet_sys, r, world, qs, ct)
        eg, fg = ls.edge_global, ls.face_global
        le, lf = xe[eg[0]:eg[0] + ls.edge_range[0]], xf[fg[0]:fg[0] + ls.face_range[0]]
        np.testing.assert_array_equal(_csr(ls.q) @ le, (_csr(qs) @ xe)[eg[1]:eg[2]])
        np.testing.assert_array_equal(_csr(ls.ct) @ lf, (_csr(ct) @ xf)[eg[1]:eg[2]])
        np.testing.assert_array_equal(_csr(ls.c) @ le, (_csr(tet_sys.c) @ xe)[fg[1]:fg[2]])
        np.testing.assert_array_equal(_csr(ls.m2) @ lf, (_csr(tet_sys.m2) @ xf)[fg[1]:fg[2]])
        owned_e.append(eg[1:])
        owned_f.append(fg[1:])
        if r > 0:  # halo below == upper end of the previous rank's owned range
            assert ls.edge_range[1] == prev.edge_range[4] and ls.face_range[1] == prev.face_range[4]
            assert prev.edge_range[0] - prev.edge_range[2] == ls.edge_range[3]
        prev = ls
    for owned, total in ((owned_e, tet_sys.n1), (owned_f, tet_sys.n2)):
        assert owned[0][0] == 0 and owned[-1][1] == total
        assert all(owned[i][1] == owned[i + 1][0] for i in range(world - 1))


def _tet_worker(rank, world, port, out):
    """One merged Strang step per rank on CPU: local rows + gloo halo exchange
    (the host logic the NCCL path runs), compared with the global step."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    sys_ = configs.tet_system(6, 0.1, seed=3)
    ls = partition.slab_system(sys_, rank, world)
    q, ct, c, m2 = (_csr(a) for a in (ls.q, ls.ct, ls.c, ls.m2))
    rng = np.random.default_rng(1)
    e_g, b_g = rng.standard_normal(sys_.n1), rng.standard_normal(sys_.n2)
    er, fr = ls.edge_range, ls.face_range
    eg, fg = ls.edge_global, ls.face_global
    e = e_g[eg[0]:eg[0] + er[0]].copy()
    b = b_g[fg[0]:fg[0] + fr[0]].copy()
    t, u = np.zeros(er[0]), np.zeros(fr[0])

    def exch(v, rngv):
        ln, lo, hi, first, last = (int(x) for x in rngv)
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(v[lo:lo + first].copy()), rank - 1))
            buf = torch.zeros(lo, dtype=torch.float64)
            dist.recv(buf, rank - 1)
            v[:lo] = buf.numpy()
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(v[hi - last:hi].copy()), rank + 1))
            buf = torch.zeros(ln - hi, dtype=torch.float64)
            dist.recv(buf, rank + 1)
            v[hi:] = buf.numpy()
        for rq in reqs:
            rq.wait()

    dt = 0.01
    o = lambda rr: slice(int(rr[1]), int(rr[2]))
    exch(e, er); t[o(er)] = q @ e; exch(t, er); b[o(fr)] -= 0.5 * dt * (c @ t)
    exch(b, fr); u[o(fr)] = m2 @ b; exch(u, fr); e[o(er)] += dt * (ct @ u)
    exch(e, er); t[o(er)] = q @ e; exch(t, er); b[o(fr)] -= 0.5 * dt * (c @ t)
    got = [None] * world
    dist.all_gather_object(got, (eg, fg, e[o(er)].tolist(), b[o(fr)].tolist()))
    if rank == 0:
        qg, cg, m2g = _csr(S.symmetric_part(sys_.q)), _csr(sys_.c), _csr(sys_.m2)
        bb = b_g - 0.5 * dt * (cg @ (qg @ e_g))
        ee = e_g + dt * (cg.T @ (m2g @ bb))
        bb = bb - 0.5 * dt * (cg @ (qg @ ee))
        err = 0.0
        for egr, fgr, el, bl in got:
            err = max(err, np.max(np.abs(np.array(el) - ee[egr[1]:egr[2]])),
                      np.max(np.abs(np.array(bl) - bb[fgr[1]:fgr[2]])))
        out.put(err)
    dist.destroy_process_group()


def test_tet_partitioned_step_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tet_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    err = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_tet_partition_lockstep_bitwise_equals_single(tet_sys, world):
    b0, e0, _ = configs.initial_pulse(tet_sys, seed=2)
    dt = 0.003
    one = S.SplitScheme(S.SplitKind.Strang, dt, tet_sys.q, tet_sys.c, tet_sys.m2, warn_cfl=False)
    ref = one.advance(S.make_state(S.Formulation.BE, b0, e0), 25)
    qs, ct = S.symmetric_part(tet_sys.q), S.transpose(tet_sys.c)
    parts = [partition.TetPart(partition.slab_system(tet_sys, r, world, qs, ct), dt)
             for r in range(world)]
    for p in parts:
        p.load_global(b0, e0)
    partition.advance_local(parts, 25)
    b, e = np.zeros(tet_sys.n2), np.zeros(tet_sys.n1)
    for p in parts:
        p.fetch_into(b, e)
    assert np.array_equal(b, ref.first) and np.array_equal(e, ref.e)
    assert partition.energy_local(parts) == pytest.approx(one.energy(ref), rel=1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_tet_device_slabs_bitwise_equal_single_device(world):
    """Slabs assembled and row-sliced on the device (the multi-GPU bench
    setup): same ranges as the host slicing, the single-GPU dt bitwise, the
    initial b = C a from local potentials, and 20 lockstep steps bitwise the
    single-GPU device scheme."""
    from paper_2301_01753_b200 import inputs
    n, jit, seed = 7, 0.1, 2023
    # the sliced-layout step (the SELL slabs' kernels; the lattice step and its
    # slabs are tests/test_gpu_slabs.py)
    one = S.tet_device_scheme(n, jit, seed=seed, dt=1.0, with_div=False, layout="sell")
    dt = configs.cfl_dt(one)
    one.set_dt(dt)
    parts = [partition.TetPart.from_device(n, jit, seed, r, world) for r in range(world)]
    sys_ = configs.tet_system(n, jit, seed=seed)
    a = inputs.gaussian(7, one._n1)
    b0 = one.apply("c", a)
    e0 = np.zeros(one._n1)
    for r, p in enumerate(parts):
        assert p.dt == dt
        assert (p.ls.n1, p.ls.n2) == (one._n1, one._n2)
        ls = partition.slab_system(sys_, r, world)
        assert np.array_equal(p.ls.edge_range, ls.edge_range)
        assert np.array_equal(p.ls.face_range, ls.face_range)
        assert p.ls.edge_global == ls.edge_global and p.ls.face_global == ls.face_global
        eg, er, fg = p.ls.edge_global, p.ls.edge_range, p.ls.face_global
        assert np.array_equal(p.apply("c", a[eg[0]:eg[0] + er[0]]), b0[fg[1]:fg[2]])
        p.load_global(b0, e0)
    ref = one.advance(S.make_state(S.Formulation.BE, b0, e0), 20)
    partition.advance_local(parts, 20)
    b, e = np.zeros(one._n2), np.zeros(one._n1)
    for p in parts:
        p.fetch_into(b, e)
    assert np.array_equal(b, ref.first) and np.array_equal(e, ref.e)
    assert partition.energy_local(parts) == pytest.approx(one.energy(ref), rel=1e-13)
    t = parts[0].kernel_timing(True)
    assert set(t) == set(partition.TetPart.KERNEL_CLASSES)


def _p2_bases(mesh):
    _, ev, fv, tv = mesh.geometry()
    e1, k1 = mesh.p2_dofs(1)
    e2, k2 = mesh.p2_dofs(2)
    b1 = np.where(k1 & 1, fv[np.minimum(e1, len(fv) - 1), 0], ev[np.minimum(e1, len(ev) - 1), 0])
    b2 = np.where(k2 & 1, tv[np.minimum(e2, len(tv) - 1), 0], fv[np.minimum(e2, len(fv) - 1), 0])
    return b1, b2


def test_p2_two_plane_halo_slabs_reproduce_global_rows():
    """Config 4's Q has the S(M1^2) pattern, which reaches two vertex planes:
    with halo = 2 the slab operators reproduce the global rows exactly, with
    halo = 1 slicing must refuse (a row would leave the halo). M1^2 stands in
    for Q here (same pattern; the host SPAI is too slow for the CPU suite)."""
    from types import SimpleNamespace
    import scipy.sparse as sp
    n, world = 5, 2
    mesh = S.TetMesh(n, 0.1, 5)
    c, m1, m2 = mesh.p2_operator("c"), mesh.p2_operator("m1"), mesh.p2_operator("m2")
    M1 = _csr(m1)
    Q = (M1 @ M1).tocsr()
    Q.sort_indices()
    q = S.SparseOperator(Q.shape[0], Q.shape[1], Q.indptr.astype(np.int64),
                         Q.indices.astype(np.int32), Q.data.copy(), True)
    sys_ = SimpleNamespace(mesh=mesh, q=q, c=c, m2=m2)
    bases = _p2_bases(mesh)
    ct = S.transpose(c)
    rng = np.random.default_rng(2)
    xe, xf = rng.standard_normal(c.cols), rng.standard_normal(c.rows)
    for r in range(world):
        ls = partition.slab_system(sys_, r, world, q, ct, halo=2, bases=bases)
        eg, fg = ls.edge_global, ls.face_global
        le, lf = xe[eg[0]:eg[0] + ls.edge_range[0]], xf[fg[0]:fg[0] + ls.face_range[0]]
        np.testing.assert_array_equal(_csr(ls.q) @ le, (Q @ xe)[eg[1]:eg[2]])
        np.testing.assert_array_equal(_csr(ls.c) @ le, (_csr(c) @ xe)[fg[1]:fg[2]])
        np.testing.assert_array_equal(_csr(ls.ct) @ lf, (_csr(ct) @ xf)[eg[1]:eg[2]])
        np.testing.assert_array_equal(_csr(ls.m2) @ lf, (_csr(m2) @ xf)[fg[1]:fg[2]])
    with pytest.raises(ValueError):
        partition.slab_system(sys_, 0, world, q, ct, halo=1, bases=bases)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_p2_device_slabs_bitwise_equal_single_device(world):
    """Config-4 slabs (two-plane halo) built on the device, 15 lockstep steps:
    bitwise the single-GPU P2 device scheme."""
    from paper_2301_01753_b200 import inputs
    n, jit, seed = 5, 0.1, 2023
    one = S.p2_device_scheme(n, jit, seed, dt=1.0, with_div=False)
    dt = configs.cfl_dt(one)
    one.set_dt(dt)
    parts = [partition.TetPart.from_device(n, jit, seed, r, world, order=2) for r in range(world)]
    a = inputs.gaussian(7, one._n1)
    b0 = one.apply("c", a)
    e0 = np.zeros(one._n1)
    for p in parts:
        assert p.dt == dt
        eg, er, fg = p.ls.edge_global, p.ls.edge_range, p.ls.face_global
        assert np.array_equal(p.apply("c", a[eg[0]:eg[0] + er[0]]), b0[fg[1]:fg[2]])
        p.load_global(b0, e0)
    ref = one.advance(S.make_state(S.Formulation.BE, b0, e0), 15)
    partition.advance_local(parts, 15)
    b, e = np.zeros(one._n2), np.zeros(one._n1)
    for p in parts:
        p.fetch_into(b, e)
    assert np.array_equal(b, ref.first) and np.array_equal(e, ref.e)
    assert partition.energy_local(parts) == pytest.approx(one.energy(ref), rel=1e-13)


@pytest.mark.gpu
def test_nccl_binding_selftest():
    """The run-time NCCL binding the slab paths use (nccl_loader.hpp): unique
    id, communicator, grouped send/recv, destroy -- on one device (1 rank)."""
    import ctypes as C
    from paper_2301_01753_b200 import _lib as L
    err = C.c_double(-1.0)
    L.check(L.lib().sfeec_nccl_selftest(0, 1 << 20, C.byref(err)))
    assert err.value == 0.0
    assert len(S.nccl_unique_id()) == 128
