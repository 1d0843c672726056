"""Inter-kernel gap of the Yee sweep: whole advance(K) vs the sum of its kernels."""
import ctypes
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2301_01753_b200 import _lib as L  # noqa: E402

R = bench.YeeRunner(bench.CONFIGS["yee256"], 0)
st = torch.cuda.current_stream()
R.set_stream(st.cuda_stream)
R.load()
R.advance(5)
torch.cuda.synchronize()
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    R.advance(200)
    b.record(st)
    torch.cuda.synchronize()
    tot = a.elapsed_time(b)
    R.timing(True)
    R.advance(200)
    ms, n = R.timing(False)
    print(f"advance(200): {tot / 200 * 1e3:.1f} us/step; kernels {ms / n * 1e3:.1f} us avg over {n}")
