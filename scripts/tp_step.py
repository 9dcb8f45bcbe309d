"""cfg 4 step times: Llama-3.1-70B (or any ARCHS model) tensor-parallel over the ranks of a
torchrun job (one process per GPU), random-init shards of the real shapes.

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 scripts/tp_step.py [--ar nccl|peer|push]
             [--B 32,64,128] [--ctx 2560] [--T 2048]
    python scripts/tp_step.py            # world 1 (NCCL identity all-reduce)

Per rank: one prefill chunk of T tokens and one CUDA-graph decode step per batch, timed
with CUDA events on the rank's stream; the JSON line (rank 0) reports the max over ranks,
decode tokens/s and the per-rank HBM bytes of a decode step (weight shard + KV shard).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11822_b200 import ops  # noqa: E402
from paper_2601_11822_b200.model import PAGE, DecoderWeights, Runner  # noqa: E402
from paper_2601_11822_b200.specs import ARCHS  # noqa: E402
from paper_2601_11822_b200.tp import IpcPeerGroup, NcclPhaseComms, local_arch, nccl_unique_id  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3.1-70b")
    ap.add_argument("--ar", default="nccl", choices=["nccl", "peer", "push"],
                    help="nccl | peer (one-shot pull all-reduce) | push (GEMM epilogue stores into every rank)")
    ap.add_argument("--B", default="32,64,128")
    ap.add_argument("--ctx", type=int, default=2560)
    ap.add_argument("--T", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29577")
        dist.init_process_group("gloo", rank=0, world_size=1)
    ops.load()
    arch = ARCHS[args.model]
    la = local_arch(arch, world)
    Bs = [int(b) for b in args.B.split(",")]
    Bmax = max(Bs)
    w = DecoderWeights.random(la, device="cuda", seed=rank, embed_vocab=arch.vocab)
    nbps = (max(args.ctx, args.T) + PAGE) // PAGE + 1
    r = Runner(w, Bmax * nbps + nbps + 8, Bmax + 1, nbps, max_prefill_tokens=args.T, max_decode_batch=Bmax,
               vocab_offset=rank * la.vocab)
    r.block_table[:Bmax] = torch.arange(Bmax * nbps, dtype=torch.int32, device="cuda").view(Bmax, nbps)
    r.block_table[Bmax] = torch.arange(Bmax * nbps, Bmax * nbps + nbps, dtype=torch.int32, device="cuda")
    if args.ar == "nccl":
        ids = [nccl_unique_id(), nccl_unique_id()] if rank == 0 else [None, None]
        obj = [ids]
        dist.broadcast_object_list(obj, src=0)
        NcclPhaseComms(r, rank, world, {"pre": obj[0][0], "dec": obj[0][1]})
    else:
        IpcPeerGroup(r, rank, world, mode=2 if args.ar == "peer" else 3)
    sms = ops.device_sm_count(local)
    st = torch.cuda.Stream()
    toks = torch.randint(0, arch.vocab, (args.T,), dtype=torch.int32, device="cuda")
    d = r.dec
    d.slot[:Bmax] = torch.arange(Bmax, dtype=torch.int32, device="cuda")
    d.pos[:Bmax] = args.ctx - 1
    d.seq[:Bmax] = args.ctx

    def timed(fn):
        with torch.cuda.stream(st):
            fn()
            st.synchronize()
            ts = []
            for _ in range(args.reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                fn()
                b.record(st)
                st.synchronize()
                ts.append(a.elapsed_time(b))
        ts.sort()
        t = torch.tensor([ts[len(ts) // 2]], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    res = {"model": args.model, "tp": world, "ar": args.ar, "ctx": args.ctx}
    res["prefill_ms"] = timed(lambda: r.prefill(Bmax, toks, 0, num_sms=sms, stream=st.cuda_stream))
    res["prefill_tok_s"] = args.T / res["prefill_ms"] * 1e3
    dec = {}
    wbytes = w.nbytes() - w.embed.numel() * 2
    for B in Bs:
        with torch.cuda.stream(st):
            r.decode_body(B, num_sms=sms, max_pages=(args.ctx + PAGE - 1) // PAGE, stream=st.cuda_stream)
            st.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                r.decode_body(B, num_sms=sms, max_pages=(args.ctx + PAGE - 1) // PAGE, stream=st.cuda_stream)
        ms = timed(g.replay)
        kv = B * args.ctx * Runner.kv_bytes_per_block(la) // PAGE
        dec[B] = {"ms": round(ms, 3), "tok_s": round(B / ms * 1e3, 1),
                  "rank_hbm_gbs": round((wbytes + kv) / ms / 1e6, 1)}
        del g
    res["decode"] = dec
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
