"""Worker of the multi-process lattice-slab tests (tests/test_gpu_slabs.py):
one process = one rank, all on cuda:0, exchanging ghost planes through the
product's CUDA-IPC transport (lattice_slab.cu). Spawned by multiprocessing."""
import os
import sys


def run_rank(rank, nranks, comm_id, cfg, b_glob, e_glob, q):
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        from paper_2301_01753_b200.partition import LatticeSlab
        s = LatticeSlab(cfg["n"], cfg["jitter"], cfg["seed"], nzg=cfg["nzg"], dt=cfg["dt"],
                        rank=rank, nranks=nranks, transport="ipc", comm_id=comm_id,
                        kind=cfg["kind"])
        s.set_state(b_glob[s.f_glob:s.f_glob + s.n2], e_glob[s.e_glob:s.e_glob + s.n1])
        cfl = s.cfl_number()
        s.advance(cfg["steps"])
        en = s.energy()
        b, e, t = s.get_state()
        q.put((rank, s.e_glob, s.f_glob, b, e, t, en, cfl, s.assembled, s.planes, None))
    except Exception as ex:  # report, never hang the parent
        q.put((rank, None, None, None, None, None, None, None, None, None, repr(ex)))
