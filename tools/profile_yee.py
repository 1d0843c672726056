"""Short Yee run for ncu captures: python tools/profile_yee.py [n] [steps] [precision] [variant]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 8
variant = int(sys.argv[4]) if len(sys.argv) > 4 else 2
y, b0, e0, dt = bench.yee_setup(n, prec, 0)
y.set_variant(variant)
y.load(b0, e0)
y.advance(steps)
print("ok", y.energy())
