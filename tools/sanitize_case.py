"""Small transforms through every kernel family, for compute-sanitizer runs:
    compute-sanitizer --tool racecheck --kernel-regex kns=sfft python tools/sanitize_case.py
Checks results against the oracle so a silent race shows up as a failure too."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07264_b200 as sf  # noqa: E402
from paper_2504_07264_b200 import dist  # noqa: E402
from oracle import oracle  # noqa: E402

rng = np.random.default_rng(0)
cases = [(6, np.float32, "tma", 700), (10, np.float32, "ldg", 40), (10, np.float64, "ldg", 40),
         (8, np.float64, "tma", 300), (12, np.float32, "ldg", 5), (14, np.float32, "auto", 2),
         (14, np.float64, "auto", 2), (3, np.float64, "ldg", 100), (10, np.float64, "tma", 300)]
for m, dt, kern, b in cases:
    for algo in ("dit", "dif"):
        re = rng.standard_normal((b, 1 << m)).astype(dt)
        im = rng.standard_normal((b, 1 << m)).astype(dt)
        plan = sf.make_plan(m, algo, dtype=torch.float32 if dt == np.float32 else torch.float64, kernel=kern)
        yr, yi = sf.fft_split(torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda(), plan=plan)
        wr, wi = oracle.fft_split_c(re, im, algo)
        gr, gi = yr.cpu().numpy().astype(np.float64), yi.cpu().numpy().astype(np.float64)
        err = np.sqrt(np.sum((gr - wr) ** 2 + (gi - wi) ** 2) / np.sum(wr ** 2 + wi ** 2))
        assert err <= 1e-5 * m, (m, dt, kern, algo, err)
# the headline kernel (fp64 N = 1024 TMA, hoisted factors, partial exchange): inverse too
re = rng.standard_normal((300, 1024))
im = rng.standard_normal((300, 1024))
for algo in ("dit", "dif"):
    yr, yi = sf.fft_split(torch.from_numpy(re).cuda(), torch.from_numpy(im).cuda(), algorithm=algo, inverse=True)
    wr, wi = oracle.fft_split_c(re, im, algo, True)
    assert np.array_equal(yr.cpu().numpy(), wr) and np.array_equal(yi.cpu().numpy(), wi)
# per-stage operators
buf = sf.InterleavedBuffer(torch.from_numpy(rng.standard_normal((3, 2 << 9))).cuda(), 9)
p9 = sf.make_plan(9)
for i in range(1, 10):
    sf.twiddle_stage(buf, p9, i)
    sf.butterfly_stage(buf, i)
# interleaved
data = torch.from_numpy(rng.standard_normal((4, 2 << 10))).cuda()
buf = sf.InterleavedBuffer(data, 10)
sf.fft(sf.make_plan(10), buf)
# sharded four-step, 2 emulated ranks
m, world = 16, 2
x = rng.standard_normal(1 << m)
plans = [dist.DistPlan(m, world, r, dtype=torch.float64) for r in range(world)]
sends = []
for r, p in enumerate(plans):
    xr = torch.as_tensor(np.ascontiguousarray(dist.scatter_input(x, world, r, p.l1))).cuda().reshape(-1)
    yr, yi = torch.empty_like(xr), torch.empty_like(xr)
    p.phase(0, xr, xr, yr, yi)
    sends.append((yr, yi))
torch.cuda.synchronize()
print("sanitize case ok")
