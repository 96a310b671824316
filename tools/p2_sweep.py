"""Time one large-N exec (device-resident planes) under the current env:
python tools/p2_sweep.py M DTYPE ALGO [reps] -> one JSON line (ms per exec)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07264_b200 as sf  # noqa: E402

m, dt, algo = int(sys.argv[1]), sys.argv[2], sys.argv[3]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
kernel = os.environ.get("P2_KERNEL", "auto")
dtype = torch.float32 if dt == "f32" else torch.float64
g = torch.Generator(device="cuda").manual_seed(4)
xr = torch.randn((1, 1 << m), dtype=dtype, device="cuda", generator=g)
xi = torch.randn((1, 1 << m), dtype=dtype, device="cuda", generator=g)
yr, yi = torch.empty_like(xr), torch.empty_like(xi)
plan = sf.make_plan(m, algo, dtype=dtype, device="cuda:0", kernel=kernel)
for _ in range(3):
    sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
s = torch.cuda.current_stream()
ev[0].record(s)
for k in range(reps):
    sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
    ev[k + 1].record(s)
torch.cuda.synchronize()
ts = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(reps))
env = {k: v for k, v in os.environ.items() if k.startswith("SFFT_") or k == "P2_KERNEL"}
print(json.dumps({"m": m, "dtype": dt, "algo": algo, "kernel": plan.kernel, "env": env,
                  "ms_med": ts[len(ts) // 2], "ms_min": ts[0]}))
