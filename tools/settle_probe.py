"""Long horizon of the headline's step time: 3000 back-to-back steps (no
per-step events: one event per 100 steps), NVML SM clock / power sampled
alongside (developer tool)."""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07264_b200 as sf  # noqa: E402
import pynvml  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "f64"
dt = torch.float64 if cfgname == "f64" else torch.float32
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10
b = (1 << 28) // (1 << m)
plan = sf.make_plan(m, dtype=dt, device="cuda:0")
g = torch.Generator(device="cuda").manual_seed(2)
xr = torch.rand((b, 1 << m), dtype=dt, device="cuda", generator=g)
xi = torch.rand((b, 1 << m), dtype=dt, device="cuda", generator=g)
yr, yi = torch.empty_like(xr), torch.empty_like(xi)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.01)


th = threading.Thread(target=sampler, daemon=True)
th.start()
time.sleep(0.5)   # idle first
nblk, per = 30, 100
ev = [torch.cuda.Event(enable_timing=True) for _ in range(nblk + 1)]
s = torch.cuda.current_stream()
walls = [time.perf_counter()]
ev[0].record(s)
for k in range(nblk):
    for _ in range(per):
        sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
    ev[k + 1].record(s)
    ev[k + 1].synchronize()
    walls.append(time.perf_counter())
stop.set()
th.join()
for k in range(nblk):
    inside = [x for x in samples if walls[k] <= x[0] <= walls[k + 1]]
    sm = sorted(x[1] for x in inside)[len(inside) // 2] if inside else None
    mem = sorted(x[2] for x in inside)[len(inside) // 2] if inside else None
    pw = round(sum(x[3] for x in inside) / len(inside), 1) if inside else None
    print(json.dumps({"block": k, "ms_per_step": round(ev[k].elapsed_time(ev[k + 1]) / per, 4), "sm_mhz": sm,
                      "mem_mhz": mem, "power_w": pw}), flush=True)
