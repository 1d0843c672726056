"""Run the device S(M1^2) SPAI once on a P2 M1 (for ncu; n from argv)."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2301_01753_b200 as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
m1 = S.TetMesh(n, 0.1, 2023).p2_operator("m1")
t0 = time.perf_counter()
q, fb = S.spai_device(m1)
print(f"n={n} N1={m1.rows} nnz(Q)={len(q.val)} fallback={fb} {time.perf_counter() - t0:.3f} s")
