"""Kernel micro-benchmarks (CUDA-event timed) for the roofline table in DESIGN.md.

    python scripts/kbench.py [--quick] [--json out.json]

GEMM shapes are Llama-3.1-8B's (prefill T=1024/2048, decode B=64..256);
decode attention uses cfg-2 shapes (ctx 1152). torch.matmul (cuBLAS) is timed
beside the GEMMs as a yardstick only.
"""

import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

PEAKS = {"hbm_gbs": 6543.4, "bf16_tflops": 1643.1}
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
        PEAKS.update(json.load(f))
except OSError:
    pass


def _graph(body, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body()  # warm-up outside capture (lazy init, smem attributes, tensor-map cache)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            body()
    return g


def _time_graph(g, iters=5):
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


HOST = {}


def timeit(fn, reps=20, flush=None):
    """Device time per call (ms): `reps` launches captured in one CUDA graph, so
    host launch overhead is excluded; with `flush`, an L2-sized memset precedes
    every call and its own graph-timed cost is subtracted."""
    import time as _t

    t0 = _t.perf_counter()
    for _ in range(10):
        fn()
    HOST["last_us"] = (_t.perf_counter() - t0) / 10 * 1e6  # host cost per call (async launch)
    torch.cuda.synchronize()
    if flush is None:
        return _time_graph(_graph(fn, reps)) / reps
    both = _time_graph(_graph(lambda: (flush.zero_(), fn()), reps))
    only = _time_graph(_graph(lambda: flush.zero_(), reps))
    return (both - only) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    dev = "cuda"
    flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)  # > L2
    scratch = ops.GemmScratch(dev)
    res = {"gemm": [], "decode_attn": []}
    shapes = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
    for T in ([1024] if args.quick else [1024, 2048]):
        for name, O, K in shapes:
            x = torch.randn(T, K, device=dev).bfloat16()
            w = (torch.randn(O, K, device=dev) * 0.02).bfloat16()
            y = torch.empty(T, O, device=dev, dtype=torch.bfloat16)
            ms = timeit(lambda: ops.linear(x, w, out=y, mode=1, scratch=scratch))
            ms_cublas = timeit(lambda: torch.matmul(x, w.T, out=y))
            tf = 2 * T * O * K / ms / 1e9
            row = dict(kind="prefill", T=T, name=name, O=O, K=K, ms=ms, host_us=HOST["last_us"], tflops=tf,
                       frac=tf / PEAKS["bf16_tflops"],
                       cublas_ms=ms_cublas, cublas_tflops=2 * T * O * K / ms_cublas / 1e9)
            res["gemm"].append(row)
            print(json.dumps(row), flush=True)
    for B in ([64, 256] if args.quick else [1, 16, 64, 128, 256]):
        for name, O, K in shapes:
            x = torch.randn(B, K, device=dev).bfloat16()
            w = (torch.randn(O, K, device=dev) * 0.02).bfloat16()
            y = torch.empty(B, O, device=dev, dtype=torch.bfloat16)
            ms = timeit(lambda: ops.linear(x, w, out=y, mode=2, scratch=scratch), flush=flush)
            ms_cublas = timeit(lambda: torch.matmul(x, w.T, out=y), flush=flush)
            gbs = (O * K * 2) / ms / 1e6
            row = dict(kind="decode", B=B, name=name, O=O, K=K, ms=ms, weight_gbs=gbs, frac_hbm=gbs / PEAKS["hbm_gbs"],
                       tflops=2 * B * O * K / ms / 1e9, cublas_ms=ms_cublas)
            res["gemm"].append(row)
            print(json.dumps(row), flush=True)
    # decode attention, Llama-8B: Hq=32, Hkv=8, ctx 1152
    Hq, Hkv, D = 32, 8, 128
    for B in ([64, 256] if args.quick else [1, 16, 64, 128, 256]):
        for ctx in ([1152] if args.quick else [1152, 8256]):
            nbps = (ctx + 15) // 16
            nb = B * nbps
            cache = torch.randn(nb, 2, Hkv, 16, D, device=dev).bfloat16()
            bt = torch.randperm(nb, device=dev).int().view(B, nbps).contiguous()
            slots = torch.arange(B, dtype=torch.int32, device=dev)
            seq = torch.full((B,), ctx, dtype=torch.int32, device=dev)
            q = torch.randn(B, Hq, D, device=dev).bfloat16()
            out = torch.empty(B, Hq, D, device=dev, dtype=torch.bfloat16)
            ws = torch.zeros(B * Hq * ((nbps + 7) // 8) * (D + 2), device=dev, dtype=torch.float32)
            res_row = {}
            for sms, gs in ((148, None),) + tuple((n, n) for n in (72,)):
                pass
            ms = timeit(lambda: ops.decode_attention(q, cache, bt, slots, seq, out, num_kv_heads=Hkv, max_pages=nbps,
                                                     workspace=ws), flush=flush)
            byts = B * ctx * Hkv * D * 2 * 2
            gbs = byts / ms / 1e6
            row = dict(B=B, ctx=ctx, ms=ms, gbs=gbs, frac_hbm=gbs / PEAKS["hbm_gbs"])
            res["decode_attn"].append(row)
            print(json.dumps(row), flush=True)
            del cache
    if args.json:
        with open(args.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
