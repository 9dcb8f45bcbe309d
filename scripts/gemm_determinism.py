"""Decode (swap-AB) GEMM repeatability and the block-packed weight layout, per partition size:
y(plain) twice, y(blocked) once, each compared bit-for-bit, plus rel. L2 against fp32.

    python scripts/gemm_determinism.py [--sms 32,48,64,148]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sms", default="32,48,64,148")
ap.add_argument("--shapes", default="28672x4096,6144x4096,4096x4096,4096x14336")
ap.add_argument("--batches", default="64,128,256")
args = ap.parse_args()
ops.load()
sc = ops.GemmScratch("cuda", ws_bytes=128 << 20)
for sms in [int(s) for s in args.sms.split(",")]:
    if sms >= 148:
        st, n = torch.cuda.Stream(), 148
    else:
        gs = ops.GreenSplit(sms)
        st, n = gs.streams[0], gs.sms[0]
    for shp in args.shapes.split(","):
        O, K = (int(v) for v in shp.split("x"))
        g = torch.Generator(device="cuda").manual_seed(O + K)
        w = (torch.randn(O, K, device="cuda", generator=g) * 0.02).bfloat16()
        wb = w.view(O // 128, 128, K // 64, 64).permute(0, 2, 1, 3).contiguous().view(O, K)
        for B in [int(b) for b in args.batches.split(",")]:
            x = torch.randn(B, K, device="cuda", generator=g).bfloat16()
            torch.cuda.synchronize()  # inputs are made on the default stream, the GEMMs run on `st`
            ys = []
            for ww, mode in ((w, 2), (w, 2), (w, 2), (wb, 2 | 8)):
                ys.append(ops.linear(x, ww, mode=mode, num_sms=n, scratch=sc, stream=st))
            st.synchronize()
            ref = x.float() @ w.float().T
            rel = lambda y: ((y.float() - ref).norm() / ref.norm()).item()  # noqa: E731
            print(json.dumps({"sms": n, "O": O, "K": K, "B": B, "repeat_equal": bool(torch.equal(ys[0], ys[1]) and
                                                                                       torch.equal(ys[0], ys[2])),
                              "blocked_equal": bool(torch.equal(ys[0], ys[3])), "rel_plain": round(rel(ys[0]), 5),
                              "rel_blocked": round(rel(ys[3]), 5)}), flush=True)
