"""Per-iteration device time of the RAPID hot path on its green-context partitions.

    python scripts/step_bench.py [--B 64,128] [--ctx 1152] [--T 1023] [--decode-sms 72] [--pdl 1,0]

decode: one CUDA-graph-captured decode step (rb_decoder_forward, all layers + lm_head +
        argmax) on the decode partition; prefill: one chunk of T tokens on the prefill
        partition. Each is timed alone and with the other partition busy (the RAPID
        steady state). CUDA events on the launching (green) streams; median of reps.
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


def med(xs):
    xs = sorted(xs)
    return xs[len(xs) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", default="64,128")
    ap.add_argument("--ctx", type=int, default=1152)
    ap.add_argument("--T", type=int, default=1023)
    ap.add_argument("--decode-sms", type=int, default=72)
    ap.add_argument("--pdl", default="1,0")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--model", default="llama3.1-8b")
    ap.add_argument("--ksplit", default="1", help="decode O/down K-slice partials: 1 on (default), 0 stream-K")
    args = ap.parse_args()
    lib = ops.load()
    arch = ARCHS[args.model]
    Bs = [int(b) for b in args.B.split(",")]
    Bmax = max(Bs)
    w = DecoderWeights.random(arch, device="cuda")
    nbps = (max(args.ctx, args.T) + 16) // 16 + 1
    nblocks = Bmax * nbps + nbps + 8
    r = Runner(w, nblocks, Bmax + 1, nbps, max_prefill_tokens=max(args.T, 16), max_decode_batch=Bmax)
    r.kv.normal_()
    r.block_table[:Bmax] = torch.arange(Bmax * nbps, dtype=torch.int32, device="cuda").view(Bmax, nbps)
    r.block_table[Bmax] = torch.arange(Bmax * nbps, Bmax * nbps + nbps, dtype=torch.int32, device="cuda")
    gs = ops.GreenSplit(args.decode_sms)
    ds, ps = gs.streams
    d = r.dec
    d.slot[:Bmax] = torch.arange(Bmax, dtype=torch.int32, device="cuda")
    d.pos[:Bmax] = args.ctx - 1
    d.seq[:Bmax] = args.ctx
    ids = torch.randint(0, arch.vocab, (args.T,), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    mp = (args.ctx + 15) // 16

    def prefill():
        with torch.cuda.stream(ps):
            r.prefill(Bmax, ids, 0, num_sms=gs.sms[1], stream=ps.cuda_stream)

    out = []
    for pdl, ks in [(int(x), int(k)) for x in args.pdl.split(",") for k in args.ksplit.split(",")]:
        lib.rb_set_pdl(pdl)
        lib.rb_set_decode_ksplit(ks)
        lib.rb_set_decode_glu(int(os.environ.get("RB_DECODE_GLU", "0")))
        for B in Bs:
            with torch.cuda.stream(ds):
                r.decode_body(B, num_sms=gs.sms[0], max_pages=mp, stream=ds.cuda_stream)
            ds.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=ds):
                r.decode_body(B, num_sms=gs.sms[0], max_pages=mp, stream=ds.cuda_stream)
            ds.synchronize()
            res = {"pdl": pdl, "ksplit": ks, "B": B, "ctx": args.ctx, "T": args.T, "decode_sms": gs.sms[0], "prefill_sms": gs.sms[1]}
            for mode in ("alone", "concurrent"):
                dts, pts = [], []
                for _ in range(args.reps):
                    torch.cuda.synchronize()
                    if mode == "concurrent":
                        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        p0.record(ps)
                        prefill()
                        p1.record(ps)
                    steps = 8
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    with torch.cuda.stream(ds):
                        e0.record(ds)
                        for _ in range(steps):
                            g.replay()
                        e1.record(ds)
                    ds.synchronize()
                    ps.synchronize()
                    dts.append(e0.elapsed_time(e1) / steps)
                    if mode == "concurrent":
                        pts.append(p0.elapsed_time(p1))
                res[f"decode_ms_{mode}"] = round(med(dts), 3)
                if mode == "concurrent":
                    res["prefill_ms_concurrent"] = round(med(pts), 3)
            # prefill alone
            pts = []
            for _ in range(args.reps):
                p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                p0.record(ps)
                prefill()
                p1.record(ps)
                ps.synchronize()
                pts.append(p0.elapsed_time(p1))
            res["prefill_ms_alone"] = round(med(pts), 3)
            print(json.dumps(res), flush=True)
            out.append(res)
            del g
    lib.rb_set_pdl(1)


if __name__ == "__main__":
    main()
