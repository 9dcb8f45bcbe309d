"""RMSNorm kernel time: rows x H bf16 (graph of 20 launches)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

ops.load()
for T, H in [(192, 4096), (1023, 4096), (2048, 5120), (64, 8192)]:
    x = torch.randn(T, H, device="cuda").bfloat16()
    w = torch.randn(H, device="cuda").bfloat16()
    y = torch.empty_like(x)
    ops.rmsnorm(x, w, y, 1e-5)
    ref = (x.float() * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-5) * w.float())
    err = float((y.float() - ref).norm() / ref.norm())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            ops.rmsnorm(x, w, y, 1e-5)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 20
    print(json.dumps({"T": T, "H": H, "us": round(us, 2), "gbs": round(2 * T * H * 2 / us / 1e3, 1), "rel_err": err}))
