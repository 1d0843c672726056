"""Short tet run for ncu captures: python tools/profile_tet.py [n] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = dict(bench.CONFIGS["tet128"], n=n)
R = bench.TetRunner(cfg, 0)
R.load()
R.advance(steps)
print("ok", R.s.energy(R.s.fetch()))
