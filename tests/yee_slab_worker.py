"""Worker of the multi-process Yee-slab tests (tests/test_gpu_yee_slabs.py):
one process = one z-slab, all on cuda:0, exchanging ghost planes through the
product's CUDA-IPC transport (yee.cu exchange_ipc). Spawned by multiprocessing."""
import os
import sys


def run_rank(rank, nranks, comm_id, cfg, b_glob, e_glob, q):
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        if cfg.get("variant") is not None:
            os.environ["SFEEC_YEE_VARIANT"] = str(cfg["variant"])
        import paper_2301_01753_b200 as S
        dims = cfg["dims"]
        em, fm = S.yee_slab_dofs(*dims, rank, nranks)
        y = S.YeeSlab(*dims, *cfg["h"], cfg["dt"], rank, nranks, comm_id,
                      precision=cfg["precision"], transport="ipc")
        y.load(b_glob[fm], e_glob[em])
        y.advance(cfg["steps"])
        en = y.energy()
        b, e, t = y.fetch()
        q.put((rank, em, fm, b, e, t, en, None))
    except Exception as ex:  # report, never hang the parent
        q.put((rank, None, None, None, None, None, None, repr(ex)))
