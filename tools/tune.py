"""Kernel-variant sweep (developer tool): times every (kernel family, radix)
of the fused path on device-resident random rows and prints GB/s of the
algorithmic traffic 4*N*sizeof(real) per transform.

    python tune.py [--sizes 6,10,12] [--dtypes f32,f64] [--bytes 1073741824]
"""

import argparse
import json

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2504_07264_b200 as sf

TMA_LR = {"f32": {5: [3], 6: [3, 2], 7: [3, 4], 8: [3, 4], 9: [3, 4], 10: [4, 3, 5], 11: [4, 3], 12: [4, 3, 6]},
          "f64": {4: [2], 5: [3], 6: [3], 7: [3, 4], 8: [3, 4], 9: [3], 10: [3, 4, 5], 11: [4]}}


def time_plan(plan, xr, xi, yr, yi, iters=60, reps=3):
    """Best of `reps` windows of `iters` back-to-back transforms (ms each)."""
    for _ in range(5):
        sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            sf.fft_split(xr, xi, out=(yr, yi), plan=plan)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        best = ms if best is None else min(best, ms)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="4,5,6,7,8,9,10,11,12")
    ap.add_argument("--dtypes", default="f32,f64")
    ap.add_argument("--bytes", type=int, default=1 << 30, help="algorithmic bytes per launch")
    ap.add_argument("--algo", default="dit")
    args = ap.parse_args()
    rows = []
    for dt in args.dtypes.split(","):
        tdt = torch.float32 if dt == "f32" else torch.float64
        esz = 4 if dt == "f32" else 8
        for m in [int(s) for s in args.sizes.split(",")]:
            n = 1 << m
            b = max(1, args.bytes // (4 * n * esz))
            xr = torch.randn(b, n, dtype=tdt, device="cuda")
            xi = torch.randn(b, n, dtype=tdt, device="cuda")
            yr, yi = torch.empty_like(xr), torch.empty_like(xi)
            variants = [("ldg", lr, None) for lr in range(1, 6)
                        if lr <= m and (n >> lr) <= 1024]
            variants += [("tma", lr, None) for lr in TMA_LR[dt].get(m, [])]
            if dt == "f32":   # both settings of the up-front base factors
                variants = [(k, lr, pf) for k, lr, _ in variants for pf in (False, True)
                            if not (pf and (lr < 2 or m < 5))]
            best = None
            for kern, lr, pf in variants:
                try:
                    plan = sf.make_plan(m, args.algo, dtype=tdt, radix_log=lr, kernel=kern,
                                        prefetch_factors=pf)
                    ms = time_plan(plan, xr, xi, yr, yi)
                except Exception as e:  # report and continue the sweep
                    rows.append({"dtype": dt, "m": m, "kernel": kern, "lr": lr, "pre": pf, "error": str(e)})
                    continue
                gbs = 4 * n * esz * b / (ms / 1e3) / 1e9
                r = {"dtype": dt, "m": m, "kernel": kern, "lr": lr, "pre": pf, "batch": b, "ms": ms, "GBs": gbs}
                rows.append(r)
                if best is None or gbs > best["GBs"]:
                    best = r
            print(json.dumps({"best": best}), flush=True)
            del xr, xi, yr, yi
            torch.cuda.empty_cache()
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
