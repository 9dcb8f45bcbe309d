"""One representative decode step and one prefill chunk of Llama-3.1-8B on the
cfg-2 partitions, for ncu launch lists / full captures (profiles/).

    python scripts/profile_step.py [--B 128] [--ctx 1150] [--T 1023] [--reps 3]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402
from paper_2601_11822_b200.model import DecoderWeights, Runner  # noqa: E402
from paper_2601_11822_b200.specs import ARCHS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=128)
ap.add_argument("--ctx", type=int, default=1150)
ap.add_argument("--T", type=int, default=1023)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--decode-sms", type=int, default=72)
ap.add_argument("--what", default="both")
ap.add_argument("--no-green", action="store_true", help="full-device streams, grids sized for the partition "
                "(Nsight Compute cannot profile green-context launches)")
args = ap.parse_args()
arch = ARCHS["llama3.1-8b"]
w = DecoderWeights.random(arch, device="cuda")
nbps = (max(args.ctx, args.T) + 16) // 16 + 1
nblocks = args.B * nbps + nbps + 8
r = Runner(w, nblocks, args.B + 1, nbps, max_prefill_tokens=max(args.T, 16), max_decode_batch=args.B)
r.kv.normal_()
bt = torch.arange(args.B * nbps, dtype=torch.int32, device="cuda").view(args.B, nbps)
r.block_table[: args.B] = bt
r.block_table[args.B] = torch.arange(args.B * nbps, args.B * nbps + nbps, dtype=torch.int32, device="cuda")
if args.no_green:
    class _Split:  # grid sizes of the split, ordinary streams
        sms = (args.decode_sms, 148 - args.decode_sms)
    gs = _Split()
    ds, ps = torch.cuda.Stream(), torch.cuda.Stream()
else:
    gs = ops.GreenSplit(args.decode_sms)
    ds, ps = gs.streams
d = r.dec
d.slot[: args.B] = torch.arange(args.B, dtype=torch.int32, device="cuda")
d.pos[: args.B] = args.ctx - 1
d.seq[: args.B] = args.ctx
ids = torch.randint(0, arch.vocab, (args.T,), dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
ev = {}
for i in range(args.reps):
    torch.cuda.nvtx.range_push(f"rep{i}")
    if args.what in ("both", "decode"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ds)
        r.decode_body(args.B, num_sms=gs.sms[0], max_pages=(args.ctx + 15) // 16, stream=ds.cuda_stream)
        e1.record(ds)
        ev.setdefault("decode", []).append((e0, e1))
    if args.what in ("both", "prefill"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ps)
        with torch.cuda.stream(ps):
            r.prefill(args.B, ids, 0, num_sms=gs.sms[1], stream=ps.cuda_stream)
        e1.record(ps)
        ev.setdefault("prefill", []).append((e0, e1))
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
for k, v in ev.items():
    print(k, [round(a.elapsed_time(b), 3) for a, b in v], "ms")
