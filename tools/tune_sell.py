"""Time the SpMV chain per kernel for the SELL variants: python tools/tune_sell.py [n]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
R = bench.TetRunner(dict(bench.CONFIGS["tet128"], n=n), 0)
R.load()
for v, sv in (("1", "0"), ("5", "0"), ("6", "0"), ("7", "0"), ("1", "0")):
    os.environ["SFEEC_SELL_VARIANT"] = v
    os.environ["SFEEC_SELL_SVARIANT"] = sv
    R.advance(5)
    name, by, ms = R.dominant(100)
    print("variant", v, sv, {k: round(d["gbs"]) for k, d in R.per_kernel.items()}, flush=True)
