"""Per-SM ingest ceiling on green-context partitions (csrc/probe.cu): pure bulk-copy streaming
global -> shared, one CTA per SM, ring depth x chunk swept, no compute. Compare with the decode
attention kernel's GB/s per SM on the same partition (scripts/attn_bench.py).

    python scripts/ingest_probe.py [--sms 16,56,88,148] [--rings 65536:2,16384:8,32768:6,8192:24]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sms", default="16,32,56,88,148")
ap.add_argument("--rings", default="8192:8,8192:16,16384:8,32768:4,32768:6,65536:3")
ap.add_argument("--tma", default="16:4:6,16:8:3,16:4:12,64:1:12,64:2:6,128:1:6,256:1:3",
                help="tensor-TMA rings box_rows:boxes_per_stage:stages")
ap.add_argument("--gb", type=float, default=4.0)
args = ap.parse_args()
lib = ops.load()
nbytes = int(args.gb * (1 << 30))
buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
sink = torch.zeros(1, dtype=torch.int32, device="cuda")
for sm in (int(s) for s in args.sms.split(",")):
    if sm >= 148:
        st, n = torch.cuda.Stream(), 148
    else:
        gs = ops.GreenSplit(sm)
        st, n = gs.streams[0], gs.sms[0]
    rings = [("bulk", r) for r in args.rings.split(",") if r] + [("tma", r) for r in args.tma.split(",") if r]
    for kind, ring in rings:
        f = [int(x) for x in ring.split(":")]
        if kind == "bulk":
            chunk, stages = f
        else:
            rows, per, stages = f
            chunk = rows * 128 * per

        def run():
            if kind == "bulk":
                rc = lib.rb_debug_stream_read(buf.data_ptr(), nbytes, chunk, stages, n, sink.data_ptr(),
                                              st.cuda_stream)
            else:
                rc = lib.rb_debug_stream_read_tma(buf.data_ptr(), nbytes, rows, per, stages, n, sink.data_ptr(),
                                                  st.cuda_stream)
            assert rc == 0, lib.rb_last_error()

        run()
        st.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(3):
            run()
        b.record(st)
        st.synchronize()
        us = a.elapsed_time(b) * 1e3 / 3
        gbs = nbytes / us / 1e3
        print(json.dumps({"sms": n, "kind": kind, "op_bytes": chunk if kind == "bulk" else rows * 128,
                          "chunk": chunk, "stages": stages, "ring_kb": chunk * stages // 1024,
                          "gbs": round(gbs, 1), "gbs_per_sm": round(gbs / n, 1)}), flush=True)
