"""Decode attention (K3) on a green-context partition: achieved HBM GB/s.

    python scripts/attn_bench.py [--sms 64,72,148] [--B 64,128,192,256] [--ctx 1152]

KV bytes per launch (K+V bf16 of one layer) exceed L2 for B >= 32, so launches stream
from HBM back to back (CUDA graph of `reps` launches, events on the partition stream).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sms", default="64,72,148")
ap.add_argument("--B", default="64,128,192,256")
ap.add_argument("--ctx", type=int, default=1152)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--no-green", action="store_true", help="grid sized for --sms but launched on a full-device "
                "stream (profilable by ncu; CTAs still one per SM)")
ap.add_argument("--one-op", default="1", help="page-load forms to sweep: 1 = one 5D op per page, 0 = four boxes")
ap.add_argument("--shapes", default="0", help="ring shapes to sweep: 0 auto, 1..4 = 12x2, 8x3, 6x4, 4x6")
args = ap.parse_args()
lib = ops.load()
D = 128
Bmax = max(int(b) for b in args.B.split(","))
nbps = (args.ctx + 15) // 16
nb = Bmax * nbps * 2 + 8
cache = torch.randn(nb, 2, args.hkv, 16, D, device="cuda").bfloat16()
bt = torch.randperm(nb - 8, device="cuda")[: Bmax * nbps].int().view(Bmax, nbps)
ws = torch.zeros(Bmax * args.hq * 64 * (D + 2), dtype=torch.float32, device="cuda")
for sm in [int(s) for s in args.sms.split(",")]:
    if sm >= 148 or args.no_green:
        st, n = torch.cuda.Stream(), min(sm, 148)
    else:
        gs = ops.GreenSplit(sm)
        st, n = gs.streams[0], gs.sms[0]
    for B, one_op, shape in [(int(b), int(o), int(sh)) for b in args.B.split(",") for o in args.one_op.split(",")
                             for sh in args.shapes.split(",")]:
        lib.rb_debug_decode_kv_one_op(one_op)
        lib.rb_debug_decode_attn_shape(shape)
        q = torch.randn(B, args.hq, D, device="cuda").bfloat16()
        out = torch.empty_like(q)
        slots = torch.arange(B, dtype=torch.int32, device="cuda")
        seq = torch.full((B,), args.ctx, dtype=torch.int32, device="cuda")

        def body():
            ops.decode_attention(q, cache, bt, slots, seq, out, num_kv_heads=args.hkv, max_pages=nbps,
                                 workspace=ws, num_sms=n, stream=st)

        with torch.cuda.stream(st):
            body()
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(args.reps):
                body()
        ts = []
        with torch.cuda.stream(st):
            g.replay()
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                g.replay()
                b.record(st)
                st.synchronize()
                ts.append(a.elapsed_time(b) * 1e3 / args.reps)
        ts.sort()
        us = ts[len(ts) // 2]
        byts = B * args.ctx * args.hkv * D * 2 * 2
        print(json.dumps({"sms": n, "one_op": one_op, "shape": shape, "B": B, "ctx": args.ctx, "us": round(us, 2), "gbs": round(byts / us / 1e3, 1)}),
              flush=True)
