"""Measure pinned H2D, D2H and concurrent H2D+D2H bandwidth (developer tool)."""
import json
import torch

n = 256 << 20  # floats = 1 GiB
h1 = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


gb = n * 4 / 1e9
t_h2d = timed(lambda: d1.copy_(h1, non_blocking=True))
t_d2h = timed(lambda: h2.copy_(d2, non_blocking=True))
t_both = timed(both)
print(json.dumps({"h2d_GBs": gb / t_h2d * 1e3, "d2h_GBs": gb / t_d2h * 1e3,
                  "concurrent_total_GBs": 2 * gb / t_both * 1e3}))
