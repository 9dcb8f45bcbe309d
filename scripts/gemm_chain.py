"""Decode GEMMs as they run inside a decode step: a CUDA-graph chain of N launches, each on a
different weight matrix (so every launch streams its weights from HBM), PDL on.

    python scripts/gemm_chain.py [--sms 72] [--batches 32,128,256] [--n 8]

Prints per-launch us and weight TB/s for our kernel and for cuBLAS (torch.matmul) in the
same chain shape, on the same green-context partition.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}


def chain_time(fn_list, stream, reps=5):
    with torch.cuda.stream(stream):
        for f in fn_list:
            f()
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for f in fn_list:
            f()
    ts = []
    with torch.cuda.stream(stream):
        g.replay()
        stream.synchronize()
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            stream.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sms", type=int, default=72)
    ap.add_argument("--batches", default="32,128,256")
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--shapes", default="qkv,o,gate_up,down")
    ap.add_argument("--variant", type=int, default=-1)
    ap.add_argument("--pair", type=int, default=-1, help="-1 auto, 0 single CTA, 1 CTA pair")
    ap.add_argument("--ksplit", default="0", help="K-slice unit counts to sweep (0 = the default schedule)")
    ap.add_argument("--blocked", action="store_true", help="weights block-packed ([O/128][K/64][128][64], one "
                    "16 KB contiguous TMA box per k-block) and launched with mode 2 | 8")
    ap.add_argument("--no-green", action="store_true", help="grid sized for --sms on a full-device stream "
                    "(profilable by ncu)")
    ap.add_argument("--pf", default="-1", help="weight L2 lookahead k-blocks to sweep (-1 auto, 0 off)")
    args = ap.parse_args()
    lib = ops.load()
    lib.rb_debug_gemm_variant(args.variant)
    lib.rb_debug_gemm_pair_mode(args.pair)
    if args.sms >= 148 or args.no_green:
        st, sms = torch.cuda.Stream(), min(args.sms, 148)
    else:
        gs = ops.GreenSplit(args.sms)
        st, sms = gs.streams[0], gs.sms[0]
    sc = ops.GemmScratch("cuda", ws_bytes=128 << 20)
    for name in args.shapes.split(","):
        O, K = SHAPES[name]
        ws = [(torch.randn(O, K, device="cuda") * 0.02).bfloat16() for _ in range(args.n)]
        mode = 2
        if args.blocked:
            plain = ws
            ws = [w.view(O // 128, 128, K // 64, 64).permute(0, 2, 1, 3).contiguous().view(O, K) for w in plain]
            mode = 2 | 8
            xc = torch.randn(128, K, device="cuda").bfloat16()
            torch.cuda.synchronize()  # made on the default stream; the GEMMs below run on `st`
            y0 = ops.linear(xc, plain[0], mode=2, num_sms=sms, scratch=sc, stream=st)
            y1 = ops.linear(xc, ws[0], mode=mode, num_sms=sms, scratch=sc, stream=st)
            st.synchronize()
            assert torch.equal(y0, y1), "blocked weights change the result"
            cub_ws = plain
        for B in [int(b) for b in args.batches.split(",")]:
            x = torch.randn(B, K, device="cuda").bfloat16()
            y = torch.empty(B, O, device="cuda", dtype=torch.bfloat16)
            ours = [lambda w=w: ops.linear(x, w, out=y, mode=mode, num_sms=sms, scratch=sc, stream=st) for w in ws]
            cub = [lambda w=w: torch.matmul(x, w.t(), out=y) for w in (cub_ws if args.blocked else ws)]
            t_cub = chain_time(cub, st) / args.n
            wb = O * K * 2
            for ks, pf in ((int(k), int(p)) for k in args.ksplit.split(",") for p in args.pf.split(",")):
                lib.rb_debug_gemm_ksplit(ks)
                lib.rb_debug_gemm_prefetch(pf)
                t_ours = chain_time(ours, st) / args.n
                lib.rb_debug_gemm_ksplit(0)
                lib.rb_debug_gemm_prefetch(-1)
                print(json.dumps({"shape": name, "B": B, "sms": sms, "blocked": args.blocked, "ksplit": ks, "pf": pf, "us": round(t_ours, 2),
                                  "tbs": round(wb / t_ours / 1e6, 2), "cublas_us": round(t_cub, 2),
                                  "cublas_tbs": round(wb / t_cub / 1e6, 2)}), flush=True)
        del ws


if __name__ == "__main__":
    main()
