"""Kernel choices of the BASELINE fp32 configs re-timed in the settled power
state (0.5 s of untimed stepping, then 200 timed steps, no idle gap):
python tools/settled_tune.py  -> one JSON line per (config, kernel, radix)
(developer tool; the AUTO table in csrc/gen_inst.py was tuned with idle gaps
between runs)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07264_b200 as sf  # noqa: E402

CASES = [
    (6, torch.float32, 1 << 20, [("tma", 3), ("tma", 2), ("ldg", 3), ("ldg", 2)]),
    (10, torch.float32, 1 << 18, [("ldg", 5), ("ldg", 4), ("ldg", 3), ("tma", 3), ("tma", 4)]),
    (12, torch.float32, 1 << 16, [("tma", 6), ("ldg", 4), ("ldg", 5), ("ldg", 3)]),
]
for m, dt, b, cands in CASES:
    n = 1 << m
    g = torch.Generator(device="cuda").manual_seed(2)
    xr = torch.rand((b, n), dtype=dt, device="cuda", generator=g)
    xi = torch.rand((b, n), dtype=dt, device="cuda", generator=g)
    yr, yi = torch.empty_like(xr), torch.empty_like(xi)
    plans = []
    for kern, lr in cands:
        try:
            plans.append((kern, lr, sf.make_plan(m, dtype=dt, device="cuda:0", kernel=kern, radix_log=lr)))
        except Exception as e:   # no such instantiation
            print(json.dumps({"m": m, "kernel": kern, "radix_log": lr, "error": str(e)[:80]}), flush=True)
    for rep in range(2):
        for kern, lr, plan in plans:
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 0.5:
                for _ in range(50):
                    sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
                torch.cuda.synchronize()
            steps = 200
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            print(json.dumps({"m": m, "kernel": kern, "radix_log": lr, "exec": plan.exec_kernel(b)[2], "ms": round(ms, 5),
                              "GBs": round(4 * n * xr.element_size() * b / ms / 1e6, 1)}), flush=True)
    del xr, xi, yr, yi
