"""One decode GEMM shape on a green-context partition, launched a few times (ncu target).

    python scripts/gemm_one.py [--sms 72] [--B 192] [--shape o] [--n 4]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
ap = argparse.ArgumentParser()
ap.add_argument("--sms", type=int, default=72)
ap.add_argument("--B", type=int, default=192)
ap.add_argument("--shape", default="o")
ap.add_argument("--n", type=int, default=4)
ap.add_argument("--residual", action="store_true")
args = ap.parse_args()
ops.load()
gs = ops.GreenSplit(args.sms)
st, sms = gs.streams[0], gs.sms[0]
sc = ops.GemmScratch("cuda")
O, K = SHAPES[args.shape]
w = (torch.randn(O, K, device="cuda") * 0.02).bfloat16()
x = torch.randn(args.B, K, device="cuda").bfloat16()
y = torch.zeros(args.B, O, device="cuda", dtype=torch.bfloat16)
for _ in range(args.n):
    ops.linear(x, w, out=y, mode=2, num_sms=sms, scratch=sc, stream=st, residual=y if args.residual else None)
torch.cuda.synchronize()
print("ok", args.shape, args.B, sms)
