"""Prefill chunk time on the prefill partition: wave-aware GEMM tile width vs fixed 256.

    python scripts/prefill_bn.py [--dsms 24,48,64,72,88] [--T 1023]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402
from paper_2601_11822_b200.model import DecoderWeights, Runner  # noqa: E402
from paper_2601_11822_b200.specs import ARCHS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dsms", default="24,48,64,72,88")
ap.add_argument("--T", type=int, default=1023)
ap.add_argument("--model", default="llama3.1-8b")
ap.add_argument("--reps", type=int, default=7)
args = ap.parse_args()
lib = ops.load()
arch = ARCHS[args.model]
w = DecoderWeights.random(arch, device="cuda")
T = args.T
r = Runner(w, 300, 4, 140, max_prefill_tokens=max(T, 2048), max_decode_batch=8)
r.block_table[1, :140] = torch.arange(140, dtype=torch.int32, device="cuda")
ids = torch.randint(0, arch.vocab, (T,), dtype=torch.int32, device="cuda")
for dsm in [int(x) for x in args.dsms.split(",")]:
    gs = ops.GreenSplit(dsm)
    ps, n = gs.streams[1], gs.sms[1]
    res = {"prefill_sms": n, "T": T}
    for bn in (256, 0):
        lib.rb_debug_gemm_prefill_bn(bn)
        ts = []
        with torch.cuda.stream(ps):
            r.prefill(1, ids, 0, num_sms=n, stream=ps.cuda_stream)
            ps.synchronize()
            for _ in range(args.reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(ps)
                r.prefill(1, ids, 0, num_sms=n, stream=ps.cuda_stream)
                b.record(ps)
                ps.synchronize()
                ts.append(a.elapsed_time(b))
        ts.sort()
        res["fixed256_ms" if bn else "auto_ms"] = round(ts[len(ts) // 2], 3)
    lib.rb_debug_gemm_prefill_bn(0)
    res["ratio"] = round(res["auto_ms"] / res["fixed256_ms"], 3)
    print(json.dumps(res), flush=True)
    del gs
