"""In-kernel timeline of a PDL chain of decode GEMM launches (absolute globaltimer).

    python scripts/gemm_chain_trace.py [--sms 64] [--B 192] [--shape o] [--n 4]

Per launch: CTA start, setup done, first / last full smem stage seen by the MMA warp,
first epilogue done, CTA end (median / max over CTAs), relative to launch 0's first CTA.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
ap = argparse.ArgumentParser()
ap.add_argument("--sms", type=int, default=64)
ap.add_argument("--B", type=int, default=192)
ap.add_argument("--shape", default="o")
ap.add_argument("--n", type=int, default=4)
ap.add_argument("--variant", type=int, default=-1)
args = ap.parse_args()
lib = ops.load()
lib.rb_debug_gemm_variant(args.variant)
gs = ops.GreenSplit(args.sms)
st, sms = gs.streams[0], gs.sms[0]
sc = ops.GemmScratch("cuda")
O, K = SHAPES[args.shape]
ws = [(torch.randn(O, K, device="cuda") * 0.02).bfloat16() for _ in range(args.n)]
x = torch.randn(args.B, K, device="cuda").bfloat16()
y = torch.empty(args.B, O, device="cuda", dtype=torch.bfloat16)
tr = torch.zeros(16 * 148 * 16, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
for _ in range(2):
    for w in ws:
        ops.linear(x, w, out=y, mode=2, num_sms=sms, scratch=sc, stream=st)
flush.zero_()
torch.cuda.synchronize()
lib.rb_debug_gemm_trace(tr.data_ptr())
for w in ws:
    ops.linear(x, w, out=y, mode=2, num_sms=sms, scratch=sc, stream=st)
torch.cuda.synchronize()
lib.rb_debug_gemm_trace(None)
t = tr.view(16, 148, 16).cpu()
t0 = t[0, :, 0][t[0, :, 0] > 0].min()
names = ["start", "setup", "mma_first_full", "mma_last_full", "epi_tfull", "epi_done", "end", "c_stored", "c_published", "f_in", "f_done", "c0_start", "c1_start", "c1_tmem", "c1_done", "c1_staged"]
print(f"{args.shape} B={args.B} sms={sms}: O={O} K={K}, weights {O * K * 2 / 1e6:.1f} MB per launch")
for i in range(args.n):
    row = t[i]
    used = row[:, 0] > 0
    r = (row[used] - t0).float() / 1000.0
    cells = []
    for j, nm in enumerate(names):
        col = r[:, j][row[used][:, j] > 0]
        if col.numel():
            cells.append(f"{nm} {col.min():6.2f}/{col.median():6.2f}/{col.max():6.2f}")
    print(f"launch {i} ({int(used.sum())} ctas): " + "  ".join(cells))
