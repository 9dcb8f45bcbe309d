"""Decode (swap-AB) GEMM probe on a real green-context partition.

    python scripts/dgemm_probe.py [--sms 72] [--batches 16,64,128,256] [--variants auto,pair]

For each Llama-3.1-8B projection and batch, times our kernel and torch.matmul (cuBLAS) on
the SAME partition stream, CUDA-graph captured, with an L2 flush before every call
(weights stream from HBM, as in a decode step). Prints one JSON row per (shape, batch).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402


def graph_time(body, stream, flush, reps=10, iters=5):
    def capture(fn):
        with torch.cuda.stream(stream):
            fn()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(reps):
                fn()
        return g

    def t(g):
        # replay() launches on the CURRENT stream: make it the partition's stream
        with torch.cuda.stream(stream):
            g.replay()
            stream.synchronize()
            ts = []
            for _ in range(iters):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                g.replay()
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b))
        ts.sort()
        return ts[len(ts) // 2]

    both = t(capture(lambda: (flush.zero_(), body())))
    only = t(capture(lambda: flush.zero_()))
    return (both - only) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sms", type=int, default=72)
    ap.add_argument("--batches", default="16,64,128,256")
    ap.add_argument("--variants", default="auto")
    ap.add_argument("--mode", type=int, default=2, help="2 = decode swap-AB (batches = B); 1 = prefill (batches = T)")
    args = ap.parse_args()
    dev = torch.device("cuda", torch.cuda.current_device())
    lib = ops.load()
    gs = None
    if args.sms < ops.device_sm_count(dev.index):
        gs = ops.GreenSplit(args.sms)
        stream, sms = gs.streams[0], gs.sms[0]
    else:
        stream, sms = torch.cuda.Stream(), ops.device_sm_count(dev.index)
    sc = ops.GemmScratch(dev)
    flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)
    shapes = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
    tot = {}
    for B in [int(b) for b in args.batches.split(",")]:
        for name, O, K in shapes:
            x = torch.randn(B, K, device=dev).bfloat16()
            w = (torch.randn(O, K, device=dev) * 0.02).bfloat16()
            y = torch.empty(B, O, device=dev, dtype=torch.bfloat16)
            ref = x.float() @ w.float().T
            row = dict(B=B, name=name, O=O, K=K, sms=sms)
            wp = w.view(O // 128, 128, K // 64, 64).permute(0, 2, 1, 3).contiguous().view(O, K)
            for var in args.variants.split(","):
                toks = set(var.split("+"))
                lib.rb_debug_gemm_pair_mode(1 if "pair" in toks else -1)
                bits = {"mt2": 1, "sk": 2, "pf": 4, "nomma": 8, "noload": 16}
                v = sum(b for k, b in bits.items() if k in toks)
                for tk in toks:
                    if tk.startswith("st"):
                        v |= int(tk[2:]) << 5
                    if tk.startswith("ka"):
                        v |= {1: 0, 2: 1, 4: 2, 8: 3}[int(tk[2:])] << 9
                lib.rb_debug_gemm_variant(-1 if "auto" in toks else v)
                mode = args.mode | (8 if "blk" in toks else 0)
                wv = wp if "blk" in toks else w
                y.fill_(float("nan"))
                torch.cuda.synchronize()
                with torch.cuda.stream(stream):
                    ops.linear(x, wv, out=y, mode=mode, num_sms=sms, scratch=sc, stream=stream)
                stream.synchronize()
                err = float((y.float() - ref).norm() / ref.norm())
                ms = graph_time(lambda: ops.linear(x, wv, out=y, mode=mode, num_sms=sms, scratch=sc, stream=stream),
                                stream, flush)
                row[f"{var}_us"] = round(ms * 1e3, 2)
                row[f"{var}_tbs"] = round(O * K * 2 / ms / 1e9, 2)
                row[f"{var}_tflops"] = round(2 * B * O * K / ms / 1e9)
                if err > 1e-2:
                    row[f"{var}_err"] = float(f"{err:.2e}")
                tot[(B, var)] = tot.get((B, var), 0.0) + ms * 1e3
            lib.rb_debug_gemm_pair_mode(-1)
            lib.rb_debug_gemm_variant(-1)
            ms = graph_time(lambda: torch.matmul(x, w.T, out=y), stream, flush)
            row["cublas_us"] = round(ms * 1e3, 2)
            row["cublas_tflops"] = round(2 * B * O * K / ms / 1e9)
            row["cublas_tbs"] = round(O * K * 2 / ms / 1e9, 2)
            tot[(B, "cublas")] = tot.get((B, "cublas"), 0.0) + ms * 1e3
            print(json.dumps(row), flush=True)
    print(json.dumps({"per_layer_us": {f"B{b}_{v}": round(t, 1) for (b, v), t in tot.items()}}), flush=True)
    if gs is not None:
        gs.close()


if __name__ == "__main__":
    main()
