"""Time the Yee sweep variants at 256^3: python tools/tune_yee.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2301_01753_b200 import _lib as L  # noqa: E402

for prec in (8, 4):
    y, b0, e0, dt = bench.yee_setup(256, prec, 0)
    for v in (2, 3, 2, 3):
        y.set_variant(v)
        y.load(b0, e0)
        y.advance(20)
        L.check(L.lib().sfeec_yee_kernel_timing(y.handle, 1, None, None))
        y.advance(300)
        ms, n = ctypes.c_double(), ctypes.c_int64()
        L.check(L.lib().sfeec_yee_kernel_timing(y.handle, 0, ms, n))
        avg = ms.value / n.value
        print(f"prec {prec} variant {v}: {avg * 1e3:.1f} us/launch, "
              f"{y.step_bytes() / (avg * 1e-3) / 1e9:.0f} GB/s", flush=True)
