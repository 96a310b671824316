"""Where does the headline's run-to-run spread come from?  One process:
several fresh allocations of the cfg3 fp64 planes (shifted by a dummy
allocation), 200 steps each with per-step CUDA events; prints per-allocation
quantiles and the series in blocks of 20 steps (developer tool)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07264_b200 as sf  # noqa: E402

b, n = 1 << 18, 1024
plan = sf.make_plan(10, dtype=torch.float64, device="cuda:0")
keep = []
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    if trial:
        keep.append(torch.empty((trial * 37 + 1) << 20, dtype=torch.uint8, device="cuda"))   # shift the next allocations
    g = torch.Generator(device="cuda").manual_seed(2)
    xr = torch.rand((b, n), dtype=torch.float64, device="cuda", generator=g)
    xi = torch.rand((b, n), dtype=torch.float64, device="cuda", generator=g)
    yr, yi = torch.empty_like(xr), torch.empty_like(xi)
    for _ in range(20):
        sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
    torch.cuda.synchronize()
    steps = 200
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    s = torch.cuda.current_stream()
    ev[0].record(s)
    for k in range(steps):
        sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
        ev[k + 1].record(s)
    torch.cuda.synchronize()
    ts = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    blocks = [round(sum(ts[i:i + 20]) / 20, 4) for i in range(0, steps, 20)]
    st = sorted(ts)
    print(json.dumps({"trial": trial, "ptr_mod_2MiB": [(t.data_ptr() >> 21) for t in (xr, xi, yr, yi)],
                      "p10": round(st[20], 4), "p50": round(st[100], 4), "p90": round(st[180], 4), "blocks": blocks}),
          flush=True)
    del xr, xi, yr, yi
    torch.cuda.empty_cache()
