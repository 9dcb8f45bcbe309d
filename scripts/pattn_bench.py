"""Prefill attention timing (graph-timed) at cfg shapes."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa
from scripts.kbench import timeit  # noqa
dev = "cuda"
for (T, start, Hq, Hkv) in [(1023, 0, 32, 8), (2048, 0, 32, 8), (2048, 6144, 40, 8), (2048, 0, 40, 8)]:
    nb = (start + T + 15) // 16 + 4
    cache = torch.randn(nb, 2, Hkv, 16, 128, device=dev).bfloat16()
    bt = torch.arange(nb, dtype=torch.int32, device=dev)
    q = torch.randn(T, Hq, 128, device=dev).bfloat16()
    out = torch.empty_like(q)
    flops = 4 * Hq * 128 * (T * T / 2 + T * start)
    row = dict(T=T, start=start, Hq=Hq, Hkv=Hkv)
    for impl in ("mma", "tc"):
        ms = timeit(lambda: ops.prefill_attention(q, cache, bt, start, out, num_kv_heads=Hkv, impl=impl))
        row[impl + "_us"] = round(ms * 1e3, 1)
        row[impl + "_tflops"] = round(flops / ms / 1e9, 1)
    print(json.dumps(row))
