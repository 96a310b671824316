"""Time the host-buffer pipeline of fft_split for several chunk sizes (developer tool)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07264_b200 as sf  # noqa: E402
from paper_2504_07264_b200 import transform  # noqa: E402

b, n = 1 << 20, 64
hr = torch.randn(b, n).pin_memory()
hi = torch.randn(b, n).pin_memory()
yr = torch.empty_like(hr).pin_memory()
yi = torch.empty_like(hi).pin_memory()
plan = sf.make_plan(6, dtype=torch.float32)
for chunk_mb in (4, 8, 16, 32, 64):
    for slots in (2, 3, 4):
        transform._PIPE_CHUNK_BYTES = chunk_mb << 20
        transform._PIPE_SLOTS = slots
        sf.fft_split(hr, hi, out=(yr, yi), plan=plan)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sf.fft_split(hr, hi, out=(yr, yi), plan=plan)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"chunk_mb": chunk_mb, "slots": slots, "ms": e0.elapsed_time(e1) / 5}), flush=True)
