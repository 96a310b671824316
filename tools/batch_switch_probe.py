"""fp64 N = 1024: the warp-per-signal kernel (radix 32) vs the radix-8 TMA
kernel by batch size, timed in the settled power state (0.5 s of untimed
stepping, then 100 timed steps, no idle gap) -- the kernel=auto batch switch
(gen_inst.py AUTO, small_below) (developer tool)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07264_b200 as sf  # noqa: E402

n = 1024
plans = {lr: sf.make_plan(10, dtype=torch.float64, device="cuda:0", kernel="tma", radix_log=lr) for lr in (3, 5)}
for lb in (12, 13, 14, 15, 16, 17):
    b = 1 << lb
    g = torch.Generator(device="cuda").manual_seed(2)
    xr = torch.rand((b, n), dtype=torch.float64, device="cuda", generator=g)
    xi = torch.rand((b, n), dtype=torch.float64, device="cuda", generator=g)
    yr, yi = torch.empty_like(xr), torch.empty_like(xi)
    for rep in range(2):
        for lr, plan in plans.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 0.5:
                for _ in range(50):
                    sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
                torch.cuda.synchronize()
            steps = 200
            e0.record()
            for _ in range(steps):
                sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            print(json.dumps({"log2_batch": lb, "radix_log": lr, "kernel": plan.exec_kernel(b)[2], "ms": round(ms, 5),
                              "GBs": round(4 * n * 8 * b / ms / 1e6, 1)}), flush=True)
