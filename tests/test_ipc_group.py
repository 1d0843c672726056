"""CPU: the shared segment and barrier under the CUDA-IPC ghost transports
(csrc/ipc_group.hpp) across real processes, world sizes 2 and 3: 200
barrier-separated rounds in which every rank writes its slot and sums all of
them. A lost or early barrier shows as a wrong sum. No GPU involved."""
import ctypes as C
import multiprocessing as mp
import os
import sys

import pytest


def _worker(rank, world, cid, rounds, q):
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        from paper_2301_01753_b200 import _lib as L
        out = C.c_double(-1.0)
        buf = (C.c_char * 128).from_buffer_copy(cid)
        L.check(L.lib().sfeec_ipc_group_selftest(C.cast(buf, C.c_void_p), rank, world, rounds,
                                                 C.byref(out)))
        q.put((rank, out.value, None))
    except Exception as ex:  # report, never hang the parent
        q.put((rank, None, repr(ex)))


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_group_rounds(world):
    from paper_2301_01753_b200.partition import ipc_unique_id
    rounds = 200
    cid = ipc_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, cid, rounds, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert not [r[2] for r in res if r[2]]
    want = sum(r + rounds - 1 for r in range(world))
    assert all(r[1] == want for r in res)
