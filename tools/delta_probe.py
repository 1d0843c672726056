"""Layout statistics of the resident tet operators (delta vs int32 columns):
python tools/delta_probe.py [n] [p2]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
p2 = len(sys.argv) > 2 and sys.argv[2] == "p2"
cfg = dict(bench.CONFIGS["p2_64" if p2 else "tet128"], n=n)
R = bench.TetRunner(cfg, 0)
for name in ("q_sym", "c", "ct", "m2"):
    print(name, R.s.layout_info(name), flush=True)
R.load()
R.advance(3)
