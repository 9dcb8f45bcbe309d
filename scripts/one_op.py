"""Run one op a few times (for ncu captures): python scripts/one_op.py gemm T O K mode | dattn B ctx"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

dev = "cuda"
kind = sys.argv[1]
if kind == "gemm":
    T, O, K, mode = map(int, sys.argv[2:6])
    x = torch.randn(T, K, device=dev).bfloat16()
    w = (torch.randn(O, K, device=dev) * 0.02).bfloat16()
    y = torch.empty(T, O, device=dev, dtype=torch.bfloat16)
    sc = ops.GemmScratch(dev)
    for _ in range(5):
        ops.linear(x, w, out=y, mode=mode, scratch=sc)
elif kind == "dattn":
    B, ctx = map(int, sys.argv[2:4])
    Hq, Hkv, D = 32, 8, 128
    nbps = (ctx + 15) // 16
    nb = B * nbps
    cache = torch.randn(nb, 2, Hkv, 16, D, device=dev).bfloat16()
    bt = torch.randperm(nb, device=dev).int().view(B, nbps).contiguous()
    slots = torch.arange(B, dtype=torch.int32, device=dev)
    seq = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    q = torch.randn(B, Hq, D, device=dev).bfloat16()
    out = torch.empty(B, Hq, D, device=dev, dtype=torch.bfloat16)
    for _ in range(5):
        ops.decode_attention(q, cache, bt, slots, seq, out, num_kv_heads=Hkv, max_pages=nbps)
torch.cuda.synchronize()
