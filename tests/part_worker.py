"""Worker of the multi-process sliced-slab tests (tests/test_gpu_part_ipc.py):
one process = one rank of partition.cu (the multi-rank path of config 4 and of
the sliced first-order kernels), all on cuda:0, halo rows pulled through the
product's CUDA-IPC transport. Spawned by multiprocessing."""
import os
import sys


def run_rank(rank, nranks, comm_id, cfg, b0, e0, q):
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        from paper_2301_01753_b200 import partition
        p = partition.TetPart.from_device(cfg["n"], cfg["jitter"], cfg["seed"], rank, nranks,
                                          order=cfg["order"])
        p.attach_ipc(comm_id)
        p.load_global(b0, e0)
        p.advance(cfg["steps"])
        en = p.energy()
        eg, fg = p.ls.edge_global, p.ls.face_global
        import numpy as np
        b, e = np.zeros(b0.size), np.zeros(e0.size)
        t = p.fetch_into(b, e)
        q.put((rank, eg, fg, b[fg[1]:fg[2]], e[eg[1]:eg[2]], t, en, p.dt, None))
    except Exception as ex:  # report, never hang the parent
        q.put((rank, None, None, None, None, None, None, None, repr(ex)))
