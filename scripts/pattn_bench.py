"""Prefill attention (K2 tcgen05) time for one chunk: T tokens after a prefix, Llama-8B heads."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

ops.load()
Hq, Hkv, D = 32, 8, 128
for T, start in [(1023, 0), (2048, 0), (2048, 6144)]:
    n = start + T
    npg = (n + 15) // 16
    cache = torch.randn(npg + 8, 2, Hkv, 16, D, device="cuda").bfloat16()
    bt = torch.arange(npg, dtype=torch.int32, device="cuda")
    q = torch.randn(T, Hq, D, device="cuda").bfloat16()
    out = torch.empty_like(q)
    for _ in range(2):
        ops.prefill_attention(q, cache, bt, start, out, num_kv_heads=Hkv)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        ops.prefill_attention(q, cache, bt, start, out, num_kv_heads=Hkv)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    fl = 4 * Hq * D * (T * T / 2 + T * start)
    print(json.dumps({"T": T, "start": start, "us": round(ms * 1e3, 1), "tflops": round(fl / ms / 1e9, 1)}))
