"""One steady-state leapfrog step of a bench config for an ncu capture of its
kernels (setup excluded via cudaProfilerStart/Stop):
ncu --profile-from-start off --set full -k regex:k_sell_pipe -c 1 ... python tools/profile_kq.py tet256"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "tet256"
R = bench.TetRunner(bench.CONFIGS[cfg], 0)
R.set_stream(torch.cuda.current_stream().cuda_stream)
R.load()
R.advance(3)
torch.cuda.synchronize()
torch.cuda.profiler.start()
R.advance(2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", cfg)
