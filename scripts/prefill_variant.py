"""Prefill chunk time on the prefill partition for GEMM schedule variants (-1 auto, 2 stream-K)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402
from paper_2601_11822_b200.model import DecoderWeights, Runner  # noqa: E402
from paper_2601_11822_b200.specs import ARCHS  # noqa: E402

lib = ops.load()
arch = ARCHS[os.environ.get("MODEL", "llama3.1-8b")]
w = DecoderWeights.random(arch, device="cuda")
T = int(os.environ.get("T", "1023"))
r = Runner(w, 300, 4, 140, max_prefill_tokens=max(T, 2048), max_decode_batch=8)
r.block_table[1, :140] = torch.arange(140, dtype=torch.int32, device="cuda")
ids = torch.randint(0, arch.vocab, (T,), dtype=torch.int32, device="cuda")
for dsm in [int(x) for x in os.environ.get("DSMS", "64,72").split(",")]:
    gs = ops.GreenSplit(dsm)
    ps, n = gs.streams[1], gs.sms[1]
    for v, (on, fr) in [(-1, (0, 0.6)), (-1, (1, 0.6)), (-1, (1, 0.35)), (-1, (1, 0.99))]:
        lib.rb_debug_gemm_variant(v)
        lib.rb_debug_gemm_prefill_streamk(on, fr)
        ts = []
        with torch.cuda.stream(ps):
            r.prefill(1, ids, 0, num_sms=n, stream=ps.cuda_stream)
            ps.synchronize()
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(ps)
                r.prefill(1, ids, 0, num_sms=n, stream=ps.cuda_stream)
                b.record(ps)
                ps.synchronize()
                ts.append(a.elapsed_time(b))
        ts.sort()
        print(json.dumps({"prefill_sms": n, "T": T, "streamk": [on, fr], "ms": round(ts[2], 3)}), flush=True)
lib.rb_debug_gemm_variant(-1)
