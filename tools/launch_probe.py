"""Host time per exec call vs device time per step (cfg2 shape)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.getcwd())
import paper_2504_07264_b200 as sf  # noqa: E402
from paper_2504_07264_b200 import _ffi  # noqa: E402

b, n = 1 << 20, 64
xr = torch.randn(b, n, device="cuda"); xi = torch.randn(b, n, device="cuda")
yr, yi = torch.empty_like(xr), torch.empty_like(xi)
plan = sf.make_plan(6, dtype=torch.float32)
sp = torch.cuda.current_stream().cuda_stream
def step():
    _ffi.lib.sfft_exec_split(plan._handle, xr.data_ptr(), xi.data_ptr(), yr.data_ptr(), yi.data_ptr(), b, n, n, -1, None, sp)
for _ in range(50): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200): step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200): step()
e1.record(); torch.cuda.synchronize()
print(f"host us/call {1e6*(t1-t0)/200:.1f}  wall us/step {1e6*(t2-t0)/200:.1f}  device us/step {1e3*e0.elapsed_time(e1)/200:.1f}")
