"""Measured B200 ARM profile (the `pdsim profile` step).

The reference's offline profiler (`pdsim profile`, cli.py:99-110; build_profile,
costmodel.py:301-335) *predicts* the smallest CU fraction whose contended decode
step fits margin x SLO for every batch of DEFAULT_BATCH_GRID. Here the same table
is MEASURED on the device: for every decode partition on the 8-SM green-context
ladder and every batch, one CUDA-graph decode step (all layers + lm_head +
argmax, the step RAPID launches) is timed on the decode green context while a
prefill chunk stream keeps the complementary partition busy. The prefill side's
chunk time under that load is recorded too, so a policy can trade decode
latency against prefill throughput.

    python -m paper_2601_11822_b200.profiler --model llama3.1-8b --ctx 1152 --out profiles/arm_llama8b.json
    python -m paper_2601_11822_b200.profiler --calibrate profiles/arm/<profile>.json --model llama3.1-8b --out fit.json

The JSON holds {"decode_us": {D: {B: us}}, "overalloc_decode_us": {B: us},
"prefill_us_per_token": {D: us}, "prefill_us_per_token_by_batch": {D: {B: us}}, ...};
`MeasuredProfile` (arm.py) reads it and
writes the reference's interchange lines `batch,fraction[,saturated]`.
"""

from __future__ import annotations

import argparse
import json
import statistics
import time

import torch

from paper_2601_11822_b200 import ops
from paper_2601_11822_b200.arm import DEFAULT_BATCH_GRID
from paper_2601_11822_b200.model import PAGE, DecoderWeights, Runner
from paper_2601_11822_b200.specs import ARCHS, SM_GRANULARITY

DEFAULT_LADDER = (16, 24, 32, 40, 48, 56, 64, 72, 88, 104, 120, 136)


def _med(xs):
    return statistics.median(xs)


def measure(model: str = "llama3.1-8b", ctx: int = 1152, chunk: int = 2048, ladder=DEFAULT_LADDER,
            batches=DEFAULT_BATCH_GRID, reps: int = 3, steps: int = 4, log=print) -> dict:
    arch = ARCHS[model]
    torch.cuda.set_device(0)
    ops.load()
    total = ops.device_sm_count(0)
    w = DecoderWeights.random(arch, device="cuda")
    nbps = (max(ctx, chunk) + PAGE) // PAGE + 1
    # batches whose KV fits next to the weights (long contexts cap the batch, as the pool would)
    free, _ = torch.cuda.mem_get_info()
    per_seq = nbps * Runner.kv_bytes_per_block(arch)
    cap = int((free - (12 << 30)) // per_seq) - 1
    batches = tuple(b for b in batches if b <= cap) or (max(1, cap),)
    Bmax = max(batches)
    nblocks = Bmax * nbps + nbps + 8
    r = Runner(w, nblocks, Bmax + 1, nbps, max_prefill_tokens=chunk, max_decode_batch=Bmax)
    r.kv.normal_(std=0.5)
    r.block_table[:Bmax] = torch.arange(Bmax * nbps, dtype=torch.int32, device="cuda").view(Bmax, nbps)
    r.block_table[Bmax] = torch.arange(Bmax * nbps, Bmax * nbps + nbps, dtype=torch.int32, device="cuda")
    d = r.dec
    d.slot[:Bmax] = torch.arange(Bmax, dtype=torch.int32, device="cuda")
    d.pos[:Bmax] = ctx - 1
    d.seq[:Bmax] = ctx
    ids = torch.randint(0, arch.vocab, (chunk,), dtype=torch.int32, device="cuda")
    mp = (ctx + PAGE - 1) // PAGE
    out = {"model": model, "ctx": ctx, "chunk": chunk, "total_sms": total, "granularity": SM_GRANULARITY,
           "batches": list(batches), "decode_us": {}, "prefill_us_per_token": {}, "prefill_alone_us_per_token": {},
           "overalloc_decode_us": {}, "overalloc_prefill_us_per_token": None}

    def run_partition(ds, ps, d_sms, p_sms):
        def prefill_chunk():
            with torch.cuda.stream(ps):
                r.prefill(Bmax, ids, 0, num_sms=p_sms, stream=ps.cuda_stream)

        # prefill alone (its chunk time sets how many chunks cover a decode window)
        prefill_chunk()
        torch.cuda.synchronize()
        pts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(ps)
            prefill_chunk()
            b.record(ps)
            ps.synchronize()
            pts.append(a.elapsed_time(b) * 1e3)
        p_alone = _med(pts)
        dec, pre_conc, pre_by_b = {}, [], {}
        for B in batches:
            with torch.cuda.stream(ds):
                r.decode_body(B, num_sms=d_sms, max_pages=mp, stream=ds.cuda_stream)
            ds.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=ds):
                r.decode_body(B, num_sms=d_sms, max_pages=mp, stream=ds.cuda_stream)
            ds.synchronize()
            g.replay()
            ds.synchronize()
            dts = []
            est = 20_000.0
            for _ in range(reps):
                torch.cuda.synchronize()
                # Both sides under load: prefill chunks and decode replays are queued on their
                # streams together, each bracketed by events; a decode step counts only if it ran
                # entirely while prefill chunks were running, and a chunk only if it ran entirely
                # inside the decode replays (an earlier version timed chunks that outlived the
                # decode window, under-stating the contention by 15-22%: profiles/r02/arm/).
                n_chunks = max(4, min(16, 1 + int(steps * est * 1.5 / max(p_alone, 1.0))))
                n_dec = max(steps, min(64, 2 + int(n_chunks * p_alone * 1.2 / max(est, 1.0))))
                ref = torch.cuda.Event(enable_timing=True)
                ref.record(ps)
                ds.wait_event(ref)
                pev, dev = [], []
                for _ in range(n_chunks):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(ps)
                    prefill_chunk()
                    b.record(ps)
                    pev.append((a, b))
                with torch.cuda.stream(ds):
                    for _ in range(n_dec):
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(ds)
                        g.replay()
                        b.record(ds)
                        dev.append((a, b))
                torch.cuda.synchronize()
                P = [(ref.elapsed_time(a) * 1e3, ref.elapsed_time(b) * 1e3) for a, b in pev]
                D = [(ref.elapsed_time(a) * 1e3, ref.elapsed_time(b) * 1e3) for a, b in dev]
                d_in = [e - s0 for s0, e in D if s0 >= P[0][0] and e <= P[-1][1]]
                p_in = [e - s0 for s0, e in P if s0 >= D[0][0] and e <= D[-1][1]]
                d_in = d_in or [e - s0 for s0, e in D]
                p_in = p_in or [e - s0 for s0, e in P]
                dts.append(_med(d_in))
                est = dts[-1]
                pre_conc.append(_med(p_in))
            dec[B] = round(_med(dts), 1)
            pre_by_b[B] = round(_med(pre_conc[-reps:]) / chunk, 3)
            del g
        return dec, _med(pre_conc) / chunk, p_alone / chunk, pre_by_b

    for D in ladder:
        t0 = time.perf_counter()
        gs = ops.GreenSplit(D)
        ds, ps = gs.streams
        dec, p_tok, p_alone_tok, p_by_b = run_partition(ds, ps, gs.sms[0], gs.sms[1])
        out["decode_us"][str(gs.sms[0])] = dec
        out.setdefault("prefill_us_per_token_by_batch", {})[str(gs.sms[0])] = p_by_b
        out["prefill_us_per_token"][str(gs.sms[0])] = round(p_tok, 3)
        out["prefill_alone_us_per_token"][str(gs.sms[0])] = round(p_alone_tok, 3)
        log(f"decode {gs.sms[0]:3d} SMs / prefill {gs.sms[1]:3d}: prefill {p_tok:.2f} us/token under load "
            f"({p_alone_tok:.2f} alone); decode us {dec}  [{time.perf_counter() - t0:.1f} s]")
    # OVERALLOCATE: both phases on the whole device, two ordinary streams
    ds, ps = torch.cuda.Stream(), torch.cuda.Stream()
    dec, p_tok, p_alone_tok, p_by_b = run_partition(ds, ps, total, total)
    out["overalloc_decode_us"] = dec
    out.setdefault("prefill_us_per_token_by_batch", {})["overalloc"] = p_by_b
    out["overalloc_prefill_us_per_token"] = round(p_tok, 3)
    out["full_prefill_alone_us_per_token"] = round(p_alone_tok, 3)
    log(f"overallocate: prefill {p_tok:.2f} us/token under load ({p_alone_tok:.2f} alone); decode us {dec}")
    return out


def calibrate_file(profile_path: str, model: str, out: str) -> dict:
    """Refit the reference cost model (GpuSpec / CostParams) to a measured profile."""
    import dataclasses

    from paper_2601_11822_b200.arm import CostParams, MeasuredProfile, calibrate
    from paper_2601_11822_b200.specs import b200_spec

    res = calibrate(MeasuredProfile.load(profile_path), ARCHS[model].model_spec(), b200_spec(), CostParams())
    res["profile"] = profile_path
    res["model"] = model
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1, default=lambda o: dataclasses.asdict(o) if dataclasses.is_dataclass(o) else o)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calibrate", default=None,
                    help="refit the reference cost model to this measured profile (no GPU needed); writes --out")
    ap.add_argument("--model", default="llama3.1-8b")
    ap.add_argument("--ctx", type=int, default=1152)
    ap.add_argument("--chunk", type=int, default=2048)
    ap.add_argument("--ladder", default=",".join(map(str, DEFAULT_LADDER)))
    ap.add_argument("--batches", default=",".join(map(str, DEFAULT_BATCH_GRID)))
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    if args.calibrate:
        r = calibrate_file(args.calibrate, args.model, args.out)
        print(json.dumps({k: r[k] for k in ("fit", "partition_decode_rel_err", "overallocate_decode_rel_err")}))
        return
    res = measure(args.model, args.ctx, args.chunk, tuple(int(x) for x in args.ladder.split(",")),
                  tuple(int(x) for x in args.batches.split(",")))
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
