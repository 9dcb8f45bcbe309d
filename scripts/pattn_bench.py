"""Prefill attention (K2 tcgen05) time for one chunk: T tokens after a prefix, Llama-8B heads,
for each CTA shape (auto / one query tile / mirrored pair of tiles).

    python scripts/pattn_bench.py [--tiles 0,1,2]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tiles", default="0,1,2")
ap.add_argument("--cases", default="1023:0,2048:0,2048:6144,512:0,1023:1024")
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--sms", type=int, default=148, help="run on the prefill side of a green-context split with this "
                "many SMs (148 = whole GPU)")
args = ap.parse_args()
lib = ops.load()
Hq, Hkv, D = args.hq, args.hkv, 128
if args.sms < 148:
    gs = ops.GreenSplit(148 - args.sms)  # first partition = the rest, second = the measured one
    st = gs.streams[1]
    assert gs.sms[1] == args.sms, gs.sms
else:
    st = torch.cuda.current_stream()
for case in args.cases.split(","):
    T, start = (int(x) for x in case.split(":"))
    n = start + T
    npg = (n + 15) // 16
    cache = torch.randn(npg + 8, 2, Hkv, 16, D, device="cuda").bfloat16()
    bt = torch.arange(npg, dtype=torch.int32, device="cuda")
    q = torch.randn(T, Hq, D, device="cuda").bfloat16()
    out = torch.empty_like(q)
    for tiles in (int(t) for t in args.tiles.split(",")):
        lib.rb_debug_pattn_tiles(tiles)
        with torch.cuda.stream(st):
            for _ in range(2):
                ops.prefill_attention(q, cache, bt, start, out, num_kv_heads=Hkv, stream=st)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(20):
                ops.prefill_attention(q, cache, bt, start, out, num_kv_heads=Hkv, stream=st)
            b.record(st)
            torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 20
        fl = 4 * Hq * D * (T * T / 2 + T * start)
        print(json.dumps({"sms": args.sms, "T": T, "start": start, "tiles": tiles, "us": round(ms * 1e3, 1),
                          "tflops": round(fl / ms / 1e9, 1)}), flush=True)
    lib.rb_debug_pattn_tiles(0)
