"""Where the Yee e2e time goes: python tools/e2e_breakdown.py [n] [steps]"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2301_01753_b200 import _lib as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
R = bench.YeeRunner(dict(bench.CONFIGS["yee256"], n=n), 0)
R.load()
R.advance(10)
pin_b = torch.from_numpy(R.b0).pin_memory()
pin_e = torch.from_numpy(R.e0).pin_memory()
out_b, out_e = torch.empty_like(pin_b).pin_memory(), torch.empty_like(pin_e).pin_memory()
dp = bench.dptr
for rep in range(3):
    t0 = time.perf_counter()
    L.check(L.lib().sfeec_yee_set_state(R.y.handle, dp(pin_b), dp(pin_e), 0.0))
    t1 = time.perf_counter()
    R.y.advance(k)
    t2 = time.perf_counter()
    L.check(L.lib().sfeec_yee_get_state(R.y.handle, dp(out_b), dp(out_e), None))
    t3 = time.perf_counter()
    print(f"set_state {1e3*(t1-t0):.2f} ms  advance({k}) {1e3*(t2-t1):.2f} ms  "
          f"get_state {1e3*(t3-t2):.2f} ms  total {1e3*(t3-t0):.2f} ms  "
          f"bytes each way {8*(R.b0.size+R.e0.size)/1e6:.0f} MB", flush=True)
# PCIe ceiling: plain pinned copies of the same byte count
nbytes = 8 * (R.b0.size + R.e0.size)
h = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"plain H2D {1e3*(t1-t0):.2f} ms ({nbytes/(t1-t0)/1e9:.1f} GB/s)  "
          f"D2H {1e3*(t2-t1):.2f} ms ({nbytes/(t2-t1)/1e9:.1f} GB/s)", flush=True)
