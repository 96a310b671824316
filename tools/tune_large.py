"""Sweep the group size limit of the multi-launch schedule (SFFT_PASS_MAX_L)
for large N: one subprocess per setting (the knob is read at plan creation)."""
import json
import os
import subprocess
import sys

CODE = r'''
import json, sys, torch
sys.path.insert(0, "%s")
import paper_2504_07264_b200 as sf
m, dt = int(sys.argv[1]), sys.argv[2]
tdt = torch.float32 if dt == "f32" else torch.float64
esz = 4 if dt == "f32" else 8
n = 1 << m
b = max(1, (1 << 30) // (4 * n * esz))
xr = torch.randn(b, n, device="cuda", dtype=tdt); xi = torch.randn_like(xr)
yr, yi = torch.empty_like(xr), torch.empty_like(xi)
plan = sf.make_plan(m, dtype=tdt)
for _ in range(5): sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
    e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 20)
print(json.dumps({"m": m, "dtype": dt, "launches": plan.launches_per_exec, "ms": best,
                  "GBs_per_step": 4 * n * esz * b / best / 1e6}))
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SIZES = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [14, 16, 18, 20, 22, 24, 26, 28]
MAXL = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [6, 7, 8, 9, 10]
for dt in sys.argv[1].split(",") if len(sys.argv) > 1 else ["f32"]:
    for m in SIZES:
        for maxl in MAXL:
            env = dict(os.environ, SFFT_PASS_MAX_L=str(maxl))
            out = subprocess.run([sys.executable, "-c", CODE, str(m), dt], env=env, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(f"maxl={maxl} {line}", flush=True)
