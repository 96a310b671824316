"""N = 2^m: per-group launches (kernel 'pass') vs L2-fused pairs ('pass2') in
the settled power state (1 s of untimed stepping, then 100 timed steps, no
idle gap): python tools/p2_settled.py M DTYPE [ALGO] (developer tool)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07264_b200 as sf  # noqa: E402

m, dtn = int(sys.argv[1]), sys.argv[2]
algo = sys.argv[3] if len(sys.argv) > 3 else "dit"
dt = torch.float32 if dtn == "f32" else torch.float64
g = torch.Generator(device="cuda").manual_seed(4)
xr = torch.randn((1, 1 << m), dtype=dt, device="cuda", generator=g)
xi = torch.randn((1, 1 << m), dtype=dt, device="cuda", generator=g)
yr, yi = torch.empty_like(xr), torch.empty_like(xi)
plans = {k: sf.make_plan(m, algo, dtype=dt, device="cuda:0", kernel=k) for k in ("pass", "pass2")}
for rep in range(3):
    for k, plan in plans.items():
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 1.0:
            for _ in range(10):
                sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
            torch.cuda.synchronize()
        steps = 100
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"m": m, "dtype": dtn, "algo": algo, "kernel": k, "ms": round(e0.elapsed_time(e1) / steps, 4)}),
              flush=True)
