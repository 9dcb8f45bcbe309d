"""What slows decode under a concurrent prefill? Decode attention (K3) on a D-SM green
context, alone and next to a background load on the other SMs:

    gemm      the prefill gate_up GEMM (T=1023, tcgen05, single-CTA tiles) back to back
    mma_only  the same GEMM with its TMA loads skipped (tensor pipe + power, no L2/HBM traffic)
    load_only the same GEMM with its MMAs skipped (TMA L2/HBM operand traffic, no tensor work)

Reports attention GB/s and the median SM clock (nvidia-smi) of each case.

    python scripts/contention_probe.py [--sms 56] [--B 224] [--ctx 1152]
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
from paper_2601_11822_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sms", default="56")
ap.add_argument("--B", type=int, default=224)
ap.add_argument("--ctx", type=int, default=1152)
ap.add_argument("--reps", type=int, default=40)
ap.add_argument("--shapes", default="0", help="decode-attention ring shapes to sweep (0 auto, 1..4 = 12x2, 8x3, 6x4, 4x6)")
ap.add_argument("--cases", default="alone,gemm,mma_only,load_only")
args = ap.parse_args()
ops.load()
lib = ops.load()
D, HQ, HKV = 128, 32, 8
B = args.B
nbps = (args.ctx + 15) // 16
nb = B * nbps + 8
cache = torch.randn(nb, 2, HKV, 16, D, device="cuda").bfloat16()
bt = torch.randperm(nb - 8, device="cuda")[: B * nbps].int().view(B, nbps)
ws = torch.zeros(B * HQ * 64 * (D + 2), dtype=torch.float32, device="cuda")
q = torch.randn(B, HQ, D, device="cuda").bfloat16()
out = torch.empty_like(q)
slots = torch.arange(B, dtype=torch.int32, device="cuda")
seq = torch.full((B,), args.ctx, dtype=torch.int32, device="cuda")
x = torch.randn(1023, 4096, device="cuda").bfloat16()
w = torch.randn(28672, 4096, device="cuda").bfloat16() * 0.02
y = torch.empty(1023, 28672, device="cuda").bfloat16()
attn_bytes = B * args.ctx * HKV * D * 2 * 2

res = []
for sm in [int(s) for s in args.sms.split(",")]:
    gs = ops.GreenSplit(sm)
    ds, ps = gs.streams
    dn, pn = gs.sms

    def attn():
        ops.decode_attention(q, cache, bt, slots, seq, out, num_kv_heads=HKV, max_pages=nbps, workspace=ws,
                             num_sms=dn, stream=ds)

    for shape in [int(v) for v in args.shapes.split(",")]:
        lib.rb_debug_decode_attn_shape(shape)
        with torch.cuda.stream(ds):
            attn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=ds):
            for _ in range(args.reps):
                attn()
        for case in args.cases.split(","):
            lib.rb_debug_gemm_pair_mode(0 if case != "gemm" else -1)
            lib.rb_debug_gemm_variant({"alone": -1, "gemm": -1, "mma_only": 16, "load_only": 8}[case])
            bg = None
            if case != "alone":
                with torch.cuda.stream(ps):
                    ops.linear(x, w, y, num_sms=pn, stream=ps)
                torch.cuda.synchronize()
                bg = torch.cuda.CUDAGraph()
                with torch.cuda.graph(bg, stream=ps):
                    for _ in range(20):
                        ops.linear(x, w, y, num_sms=pn, stream=ps)
            torch.cuda.synchronize()
            clk = ClockSampler(0)
            clk.start()
            ts, gts = [], []
            for _ in range(8):
                if bg is not None:  # graph replays launch on the CURRENT stream
                    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    with torch.cuda.stream(ps):
                        a0.record(ps)
                        bg.replay()
                        bg.replay()
                        a1.record(ps)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(ds):
                    e0.record(ds)
                    g.replay()
                    e1.record(ds)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / args.reps)
                if bg is not None:
                    gts.append(a0.elapsed_time(a1) * 1e3 / 40)
            c = clk.stop()
            us = statistics.median(ts)
            r = {"decode_sms": dn, "shape": shape, "case": case, "attn_us": round(us, 1), "attn_gbs": round(attn_bytes / us / 1e3, 1),
                 "bg_gemm_us": round(statistics.median(gts), 1) if gts else None, "sm_mhz": c.get("sm_mhz"),
                 "reasons": c.get("reasons")}
            print(json.dumps(r), flush=True)
            res.append(r)
            del bg
        lib.rb_debug_gemm_variant(-1)
        lib.rb_debug_gemm_pair_mode(-1)
        lib.rb_debug_decode_attn_shape(0)
        del g
    gs.close()
