"""Headline benchmark: RAPID-Serve on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--qps Q] [--duration S] [--model llama3.1-8b] [--slo-ms 50]
                    [--decode-sms 72 | --arm | --arm-profile PATH --arm-policy adaptive|balanced|slo-min]
                    [--engine rapid|hybrid-<chunk>] [--compare hybrid-2048|none]
                    [--prompt 1024 --output 256] [--timeline PATH]

Workload (BASELINE.json configs[2], "cfg 3", the configuration the SLO-constrained metric
is defined on): Llama-3.1-8B bf16 (random-init weights of the real shapes; no checkpoints
offline), one B200 per replica, synthetic trace `synthesize(WorkloadSpec(qps=Q*N,
duration_s=S, seed=42, mean_prompt_tokens=1024, mean_output_tokens=256, sigma=0))` with
request i served by replica i mod N (replicas.shard_items), each replica the real-time RAPID
engine (prefill and decode of different requests concurrently on disjoint SM partitions over
one shared paged KV cache) with the measured ARM (profiles/arm/; default policy per
model: "feedback" for 8B, "balanced" for Qwen-14B; tables re-measured in round 2 with both phases
strictly under load)
choosing the green-context split at every launch. `--decode-sms 72` runs cfg 2 (static
green-context 50/50 split), `--arm` the reference cost-model allocate(), `--engine
hybrid-2048` the same engine's chunked-prefill comparator as the primary arm.

value (the BASELINE metric): the reference's run-level `summarize().tokens_per_s`
(pkg/src/pdsim/metrics.py:146-200: output-token stamps in [10% of the horizon, horizon] /
that window), pooled over all replicas (whole job), and SLO-constrained: it is the rate only
when the pooled p99 ITL <= --slo-ms, else 0 (the unconstrained rate is reported beside it).
The same-engine hybrid-2048 comparator (north-star target: RAPID beats it) is served on the
SAME trace in the same invocation and reported under "comparator".

Steps: a step is one decode iteration (one CUDA-graph replay over the current batch; prefill
chunks run concurrently on the other partition). After >= W warm-up steps and the summarize
warm-up cut, exactly K steps are timed between CUDA events on the decode stream
("device_window", ms_per_step) with nvidia-smi clocks sampled during them; `e2e` is the host
wall-clock rate over the same K steps through RapidEngine/B200Executor (pinned H2D of step
inputs, block-table deltas and prefill ids, D2H of sampled ids, every step). The trace is
sized so the run holds W + K steps (>= 60 s). Inputs are larger than L2 (KV cache and
weights, ~30 GB per step), so no extra flush is needed.

roofline: decode attention (K3), measured IN SITU: CUDA events recorded around the middle
layer's attention launch inside every decode graph (rb_workspace_t.probe_ev*), summed over
the K timed steps on whatever partition the ARM chose; algorithmic bytes per launch =
sum over rows of ctx * Hkv * 128 * 2 (K,V) * 2 B. `roofline.partition_bound` puts the same
launches against min(HBM, decode SMs x 64 B x in-situ SM clock): on the small decode partitions
the SMs' shared-memory port, not HBM, bounds K3.

N > 1 (torchrun): one independent replica per GPU ("replicas only"; the path shards by
request, no data-path collective); barrier + max-over-ranks of the device window; tokens and
latency samples pooled over ranks (replicas.pool_window_stats).
"""


from __future__ import annotations

import argparse
import collections
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SLO_ITL_US = 50_000
PROMPT, OUTPUT = 1024, 256
# measured ARM tables (python -m paper_2601_11822_b200.profiler), per model, at its benchmark mix
DEFAULT_PROFILES = {"llama3.1-8b": "llama3.1-8b_ctx1152_chunk1023_r02.json", "qwen2.5-14b": "qwen2.5-14b_ctx8256_r02.json"}
# measured-ARM policy per model (same-box runs, profiles/r02/): 8B 1024/256 — feedback beats balanced by
# 3-5% (time-shares the 32/64-SM hull pair); Qwen-14B 8192/128 — balanced (32 decode SMs) 438 tok/s,
# feedback settles on 56 and starves prefill (355)
DEFAULT_POLICY = {"llama3.1-8b": "feedback", "qwen2.5-14b": "balanced"}


def _peaks() -> dict:
    p = {"hbm_gbs": 6543.4, "bf16_tflops": 1643.1, "bf16_tflops_sustained": 1381.0, "_src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p.update(json.load(fh))
            p["_src"] = "measured"
    except OSError:
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw,power.limit")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons, pw, plim = [], None, set(), [], None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
            try:
                pw.append(float(f[6]))
                plim = float(f[7])
            except (IndexError, ValueError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(pw) if pw else None, "power_limit_w": plim}


def dist_setup(backend: str = "nccl"):
    """One process per GPU. backend "gloo" (TP peer modes) also allows several ranks on one
    GPU: ranks map onto the visible devices round-robin."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        if backend == "nccl" and torch.cuda.device_count() < int(os.environ.get("LOCAL_WORLD_SIZE", world)):
            backend = "gloo"  # more ranks than GPUs (path validation on a one-GPU box): share the devices
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
    return rank, world, local


def run_reference(args, rank, world):
    """--impl reference: the CPU restatement of the path (oracle port), same metric. W warm-up and
    K timed steps, each one bounded sample of the workload (one prefill chunk + one batched
    decode step on the host's cores); the model and KV state are built once, untimed."""
    if rank != 0:
        return
    from oracle.cpu_baseline import CpuSampler
    from paper_2601_11822_b200.specs import ARCHS

    sampler = CpuSampler(ARCHS[args.model], PROMPT, OUTPUT, batch=8, prefill_tokens=32)
    for _ in range(args.warmup):
        sampler.step()
    res = [sampler.step() for _ in range(max(1, args.steps))]
    t_pref = statistics.median(r["t_prefill_per_token_s"] for r in res)
    t_dec = statistics.median(r["t_decode_per_token_s"] for r in res)
    v = 1.0 / (t_dec + (PROMPT / OUTPUT) * t_pref)
    line = {
        "impl": "reference", "metric": "SLO-constrained output tokens/s per GPU (p99 ITL<=SLO); p50 TTFT; p99 ITL",
        "value": v, "unit": "output tokens/s", "n_gpus": world, "steps": len(res), "warmup": args.warmup,
        "ms_per_step": statistics.mean(r["wall_s"] for r in res) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"cfg3 {args.model} bf16 path restated in fp32 on the host, in {PROMPT}/out {OUTPUT} "
                               f"(bounded CPU sample per step: one prefill chunk + one batched decode step)"},
        "cpu_baseline": {"value": v, "unit": "output tokens/s", "cores": sampler.threads, "kind": "port",
                         "sample": sampler.describe()},
        "e2e": {"value": v, "unit": "output tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def time_decode_attention(runner, stream, B: int, ctx: int, sms: int, iters: int = 20) -> dict:
    """Live roofline probe of the dominant decode kernel on the decode partition:
    CUDA events over `iters` launches at the run's mean (B, ctx)."""
    import torch

    from paper_2601_11822_b200 import ops

    arch = runner.arch
    nbps = (ctx + 15) // 16
    B = max(1, min(B, runner.num_slots, runner.num_blocks // max(1, nbps)))
    slots = torch.arange(B, dtype=torch.int32, device=runner.device)
    seq = torch.full((B,), ctx, dtype=torch.int32, device=runner.device)
    bt = torch.arange(B * nbps, dtype=torch.int32, device=runner.device).view(B, nbps)
    tbl = runner.block_table.clone()
    tbl[:B, :nbps] = bt
    q = torch.randn(B, arch.q_heads, arch.head_dim, device=runner.device).bfloat16()
    out = torch.empty_like(q)
    cache = runner.kv[0]
    sh = stream.cuda_stream
    for _ in range(3):
        ops.decode_attention(q, cache, tbl, slots, seq, out, num_kv_heads=arch.kv_heads, max_pages=nbps,
                             workspace=runner.attn_ws, num_sms=sms, stream=sh)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        ops.decode_attention(q, cache, tbl, slots, seq, out, num_kv_heads=arch.kv_heads, max_pages=nbps,
                             workspace=runner.attn_ws, num_sms=sms, stream=sh)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / iters
    byts = B * ctx * arch.kv_heads * arch.head_dim * 2 * 2  # K+V bf16, one layer, one launch
    return {"B": B, "ctx": ctx, "bytes": byts, "ms": ms, "gbs": byts / ms / 1e6}



def _free_cuda():
    import gc

    import torch

    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def serve(args, arch, items, horizon, engine_kind, rank, world, local, *, primary, executor=None):
    """Serve `items` with one engine on this rank's GPU; returns the measurements.
    `executor`: a prebuilt executor (rank 0 of a TP group: tp_serve.build_tp_executor)."""
    import torch

    from paper_2601_11822_b200.arm import CostParams
    from paper_2601_11822_b200.clock import RealTimeLoop
    from paper_2601_11822_b200.engines.hybrid import HybridEngine
    from paper_2601_11822_b200.engines.rapid import RapidEngine
    from paper_2601_11822_b200.executor_b200 import B200Executor, HybridB200Executor
    from paper_2601_11822_b200.harness import check_invariants
    from paper_2601_11822_b200.replicas import local_window_stats, pool_window_stats
    from paper_2601_11822_b200.slo import SloSpec
    from paper_2601_11822_b200.specs import AllocationDecision, AllocationMode, b200_spec

    hybrid = engine_kind.startswith("hybrid-")
    use_arm = args.arm or hybrid
    # engine knob max_batch (config.py:263, default 256) per arm
    mb = args.max_batch if primary else args.compare_max_batch
    max_ctx = PROMPT + OUTPUT + 64
    if hybrid:
        hchunk = int(engine_kind.split("-", 1)[1])
        ex = HybridB200Executor(arch, seed=rank, max_batch=mb, chunk_tokens=hchunk, max_context=max_ctx,
                                num_slots=4096)
    elif executor is not None:
        ex = executor
    else:
        ex = B200Executor(arch, seed=rank, static_decode_sms=None if args.arm else args.decode_sms, max_batch=mb,
                          kv_memory_fraction=args.kv_memory_fraction,
                          chunk_tokens=2048, max_context=max_ctx, num_slots=4096, probe_attention=True)
    policy = None
    if args.arm_profile and not hybrid:
        from paper_2601_11822_b200.arm import MeasuredArm, MeasuredProfile

        policy = MeasuredArm(MeasuredProfile.load(args.arm_profile), SLO_ITL_US, mb, args.arm_policy)
        ex.warmup(sorted(policy.splits_used(), key=lambda d: -1 if d is None else d))
    else:
        ex.warmup()
    pkey = None if use_arm else args.decode_sms
    total = ex.total_sms
    model = arch.model_spec()
    slo = SloSpec(itl_slo_us=SLO_ITL_US)
    if hybrid:
        engine = HybridEngine(model, b200_spec(), CostParams(), slo, chunk_tokens=hchunk, max_batch=mb, executor=ex)
    else:
        part = ex._partitions[pkey]
        static = None if args.arm else AllocationDecision(AllocationMode.PARTITION, part.p_sms / total,
                                                          part.d_sms / total)
        gpu_spec, cost_params = b200_spec(), CostParams()
        if args.arm_calibrated:  # the reference allocate() on the refitted model
            import dataclasses

            from paper_2601_11822_b200.specs import GpuSpec

            with open(args.arm_calibrated) as fh:
                fit = json.load(fh)
            gpu_spec = GpuSpec(**fit["gpu"])
            cost_params = dataclasses.replace(CostParams(), **fit["params"])
        engine = RapidEngine(model, gpu_spec, cost_params, slo, chunk_tokens=2048, max_batch=mb, executor=ex,
                             static_decision=static, record_decisions=args.arm, arm_policy=policy)

    # ---- timed window over K decode steps, hooked on the executor
    cut_us = int(0.10 * horizon)  # summarize()'s warm-up cut: the device window starts after it
    win = {"start_handle": None, "end_handle": None, "tokens": 0, "steps": 0, "host0": None, "host1": None,
           "h2d0": 0, "h2d1": 0, "d2h0": 0, "d2h1": 0, "launch0": 0, "launch1": 0, "Bs": [], "ctxs": []}
    clocks = ClockSampler(local)
    launch_name, finish_name = ("launch_hybrid", "finish_hybrid") if hybrid else ("launch_decode", "finish_decode")
    orig_launch = getattr(ex, launch_name)
    orig_finish = getattr(ex, finish_name)
    loop_ref = {}

    def launch_decode(members, *a):
        h = orig_launch(members, *a)
        st = win
        if st["start_handle"] is None and ex.decode_steps > args.warmup and loop_ref["loop"].clock_us() >= cut_us:
            st["start_handle"] = h
            st["host0"] = time.perf_counter()
            st["h2d0"], st["d2h0"], st["launch0"] = ex.h2d_bytes, ex.d2h_bytes, ex.gpu_launches
            clocks.start()  # both arms: the comparator's clocks are reported too
        if st["start_handle"] is not None and st["end_handle"] is None:
            st["steps"] += 1
            st["Bs"].append(len(members))
            if members:
                st["ctxs"].append(sum(r.context_tokens for r in members) / len(members))
            h._win = True
            if st["steps"] == args.steps:
                st["end_handle"] = h
        return h

    def finish_decode(h):
        orig_finish(h)
        if getattr(h, "_win", False):
            win["tokens"] += sum(1 for lame in h.lame if not lame)
            if h.kind == "hybrid" and getattr(h, "req", None) is not None:
                win["tokens"] += 1  # first token of the request whose prompt this chunk finished
            if h is win["end_handle"]:
                win["host1"] = time.perf_counter()
                win["h2d1"], win["d2h1"], win["launch1"] = ex.h2d_bytes, ex.d2h_bytes, ex.gpu_launches
                win["clocks"] = clocks.stop()

    setattr(ex, launch_name, launch_decode)
    setattr(ex, finish_name, finish_decode)

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    loop = RealTimeLoop(until_us=horizon, poll_sleep_us=args.poll_sleep_us)
    loop_ref["loop"] = loop
    engine.prime(loop, items)
    t_run = time.perf_counter()
    loop.run(engine.on_event)
    t_run = time.perf_counter() - t_run
    torch.cuda.synchronize()
    check_invariants(engine)
    if win.get("clocks") is None and clocks.proc is not None:
        win["clocks"] = clocks.stop()

    complete = win["end_handle"] is not None and win["host1"] is not None
    ms = win["start_handle"].ev0.elapsed_time(win["end_handle"].ev1) if complete else float("nan")
    host_s = win["host1"] - win["host0"] if complete else float("nan")
    tokens = win["tokens"]
    # in-situ decode-attention probe over the timed steps
    w0 = getattr(win["start_handle"], "launch_ns", 0) if complete else 0
    w1 = getattr(win["end_handle"], "launch_ns", 0) if complete else 0
    probe = [(b, m, s) for b, m, s, ns in getattr(ex, "attn_probe_log", []) if w0 <= ns <= w1]
    pb, pm = float(sum(b for b, _, _ in probe)), float(sum(m for _, m, _ in probe))
    by_part = collections.defaultdict(lambda: [0.0, 0.0, 0])
    for b, m, s in probe:
        by_part[s][0] += b
        by_part[s][1] += m
        by_part[s][2] += 1
    if world > 1:
        cdev = "cuda" if torch.distributed.get_backend() == "nccl" else "cpu"
        t = torch.tensor([ms, host_s, pb, pm], dtype=torch.float64, device=cdev)
        torch.distributed.all_reduce(t[:2], op=torch.distributed.ReduceOp.MAX)
        tk = torch.tensor([tokens, pb, pm], dtype=torch.float64, device=cdev)
        torch.distributed.all_reduce(tk, op=torch.distributed.ReduceOp.SUM)
        ms, host_s, tokens, pb, pm = float(t[0]), float(t[1]), float(tk[0]), float(tk[1]), float(tk[2])
    pooled = pool_window_stats(local_window_stats(engine.requests, slo, loop.horizon_us), pool=world > 1)

    steps = max(1, win["steps"])

    def duty(log, t0, t1):
        sel = [(g, ns) for g, ns in log if t0 <= ns <= t1]
        if len(sel) < 2:
            return None
        span_us = (sel[-1][1] - sel[0][1]) / 1e3
        return round(sum(g for g, _ in sel[:-1]) / span_us, 3) if span_us > 0 else None

    res = {
        "engine": engine_kind, "pooled": pooled, "complete": complete, "ms": ms, "host_s": host_s, "tokens": tokens,
        "steps": win["steps"], "clocks": win.get("clocks"),
        "h2d": (win["h2d1"] - win["h2d0"]) / steps if complete else 0,
        "d2h": (win["d2h1"] - win["d2h0"]) / steps if complete else 0,
        "launches": int(win["launch1"] - win["launch0"]) if complete else 0,
        "mean_batch": statistics.mean(win["Bs"]) if win["Bs"] else None,
        "mean_ctx": statistics.mean(win["ctxs"]) if win["ctxs"] else None,
        "probe": {"bytes": pb, "ms": pm, "launches": len(probe),
                  "by_sms": {str(k): {"gbs": v[0] / v[1] / 1e6 if v[1] else None, "launches": v[2],
                                      "bytes": v[0], "ms": v[1]}
                             for k, v in sorted(by_part.items())}},
        "host_gap": _gap_stats(getattr(ex, "host_gap_log", [])),
        "host_prof": ({k: round(v / max(1, ex.host_prof["steps"]) / 1e3, 1) for k, v in ex.host_prof.items()
                       if k != "steps"} if getattr(ex, "host_prof", None) else None),
        "duty": {"decode": duty([(g, ns) for _, g, ns in ex.step_log], w0, w1),
                 "prefill": duty(getattr(ex, "prefill_log", []), w0, w1)},
        "run_wall_s": t_run, "requests": len(engine.requests),
        "finished_all": sum(1 for r in engine.requests if r.state.value == "finished"),
        "policy": policy, "total_sms": total, "pkey": pkey,
        "arm_decisions": ({**{k: sum(1 for _, d in engine.decision_log if d.mode.value == k)
                              for k in ("overallocate", "partition")},
                           "decode_sms": dict(sorted(collections.Counter(
                               str(round(d.cu_fraction_decode * total)) for _, d in engine.decision_log
                               if d.mode.value == "partition").items()))}
                          if getattr(engine, "decision_log", None) else None),
    }
    if args.timeline and rank == 0:
        _write_timeline(args.timeline + f".{engine_kind}.json", engine, ex, loop.horizon_us)
    if primary and not hybrid:
        res["ex"], res["part"] = ex, ex._partitions[pkey]
    else:
        ex.close()
    del engine
    return res


def partition_bound(by_sms: dict, sm_mhz: float | None, hbm_gbs: float) -> dict | None:
    """K3's in-situ rate against its partition bound. Every KV byte crosses an SM's shared memory
    twice (TMA write, ldmatrix read) and one SM's shared memory moves 128 B per clock, so a d-SM
    partition streams at most d x 64 B x f_SM (profiles/r02/dattn/smem_port/); the
    bound is min(HBM, that). by_sms: {decode SMs: {"gbs", "bytes", "ms"}} of the timed launches;
    "frac" = time at the bound / measured time over all of them."""
    if not sm_mhz or not by_sms:
        return None
    t_bound = t_act = 0.0
    per = {}
    for k, v in by_sms.items():
        bound = min(hbm_gbs, int(k) * 64 * sm_mhz * 1e6 / 1e9)
        per[k] = {"bound_gbs": round(bound, 1), "frac": round(v["gbs"] / bound, 3) if v["gbs"] else None}
        if v["ms"]:
            t_bound += v["bytes"] / (bound * 1e6)
            t_act += v["ms"]
    return {"bound": "min(hbm, decode SMs x 64 B x in-situ SM clock)", "sm_mhz": sm_mhz, "by_decode_sms": per,
            "frac": round(t_bound / t_act, 3) if t_act else None}


def _tpj(m):
    """Output tokens per joule over the timed window: window tokens/s / median board power."""
    c = m.get("clocks") or {}
    if not m.get("complete") or not c.get("power_w") or not m.get("ms"):
        return None
    return round(m["tokens"] / (m["ms"] / 1e3) / c["power_w"], 3)


def _gap_stats(log):
    """Host time per decode step: from a step's completion handling to the next launch."""
    if not log:
        return None
    xs = sorted(log)
    return {"median_us": xs[len(xs) // 2], "mean_us": round(sum(xs) / len(xs), 1),
            "p99_us": xs[min(len(xs) - 1, int(0.99 * len(xs)))], "steps": len(xs)}


def _write_timeline(path, engine, ex, horizon_us):
    """Per-second diagnostics: delivered tokens, decode steps / batch, decode SMs, queue."""
    nsec = int(horizon_us // 1_000_000) + 10
    tok = [0] * nsec
    for r in engine.requests:
        for t in r.token_times_us:
            if 0 <= t // 1_000_000 < nsec:
                tok[int(t // 1_000_000)] += 1
    ttft = collections.defaultdict(list)
    for r in engine.requests:
        if r.token_times_us:
            ttft[int(r.arrival_us // 1_000_000)].append((r.token_times_us[0] - r.arrival_us) / 1e3)
    out = {"tokens_per_s": tok, "ttft_ms_by_arrival_s": {k: statistics.mean(v) for k, v in sorted(ttft.items())},
           "step_log": ex.step_log[:20000], "prefill_log": getattr(ex, "prefill_log", [])[:20000]}
    if getattr(engine, "decision_log", None):
        out["decisions"] = [(ph, round(d.cu_fraction_decode * 148)) for ph, d in engine.decision_log][:40000]
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "w") as fh:
        json.dump(out, fh)


def main():
    global PROMPT, OUTPUT, SLO_ITL_US
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # 56 QPS per replica (14.3k output tok/s offered) saturates the RAPID engine on one B200
    # with p99 ITL under the SLO: the saturated delivered rate is the SLO-constrained maximum
    ap.add_argument("--qps", type=float, default=56.0)
    ap.add_argument("--duration", type=float, default=None)
    ap.add_argument("--decode-sms", type=int, default=None,
                    help="cfg 2: static split with this many decode SMs (72 = the green-context 50/50)")
    ap.add_argument("--model", default="llama3.1-8b")
    ap.add_argument("--prompt", type=int, default=PROMPT, help="mean prompt tokens (cfg 5: 8192)")
    ap.add_argument("--output", type=int, default=OUTPUT, help="mean output tokens (cfg 5: 128)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--engine", default="rapid", help="rapid | hybrid-<chunk> (same-engine chunked-prefill comparator)")
    ap.add_argument("--compare", default="auto",
                    help="second arm on the same trace in the same run: hybrid-<chunk> | none (auto: hybrid-2048 "
                         "when --engine rapid)")
    ap.add_argument("--poll-sleep-us", type=int, default=0,
                    help="real-time loop sleep between CUDA-event polls (0 = busy-poll while GPU work is pending)")
    ap.add_argument("--tp", type=int, default=1, help="cfg 4: tensor parallel over the whole job (world == tp)")
    ap.add_argument("--tp-ar", default="nccl", choices=["nccl", "peer", "push"],
                    help="TP all-reduce: NCCL (NVLink) or the peer-memory kernels (also several ranks on one GPU)")
    ap.add_argument("--kv-memory-fraction", type=float, default=0.90,
                    help="share of free HBM the KV cache takes (the reference's 10%% rule: 0.9)")
    ap.add_argument("--max-batch", type=int, default=256, help="engine max_batch of the primary arm (config.py:263)")
    ap.add_argument("--compare-max-batch", type=int, default=256, help="max_batch of the hybrid comparator")
    ap.add_argument("--slo-ms", type=float, default=SLO_ITL_US / 1e3, help="p99 ITL SLO (default 50 ms)")
    ap.add_argument("--arm-profile", default="auto",
                    help="measured B200 ARM tables (profiler.py JSON; 'auto' = the committed profile of --model "
                         "under profiles/arm/)")
    ap.add_argument("--arm-policy", default=None, choices=["balanced", "slo-min", "adaptive", "feedback"],
                    help="measured-ARM policy (default: per model, DEFAULT_POLICY)")
    ap.add_argument("--arm", action="store_true",
                    help="the reference allocate() on the cost model instead of the measured ARM")
    ap.add_argument("--arm-calibrated", default=None,
                    help="with --arm: the reference cost model refitted to the B200 tables (profiler --calibrate JSON)")
    ap.add_argument("--timeline", default=None, help="write per-second diagnostics to PATH.<engine>.json")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    PROMPT, OUTPUT = args.prompt, args.output
    SLO_ITL_US = int(args.slo_ms * 1e3)
    if args.compare == "auto":
        args.compare = "hybrid-2048" if args.engine == "rapid" else "none"
    if args.arm_calibrated:
        args.arm = True
    if args.decode_sms is not None or args.arm or args.engine != "rapid":
        args.arm_profile = None
    elif args.arm_profile == "auto":
        args.arm_profile = os.path.join(ROOT, "profiles", "arm", DEFAULT_PROFILES.get(args.model, ""))
        if not os.path.isfile(args.arm_profile):
            args.arm_profile = None
            args.arm = True
    if args.arm_profile:
        args.arm = True
    if args.arm_policy is None:
        args.arm_policy = DEFAULT_POLICY.get(args.model, "balanced")
    if args.decode_sms is None:
        args.decode_sms = 72

    if args.tp > 1:  # cfg 4: one engine, tensor parallel over the whole job (no replicas, no comparator)
        args.compare = "none"
        args.arm = False
        args.arm_profile = None
    rank, world, local = dist_setup("gloo" if args.tp > 1 and args.tp_ar != "nccl" else "nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.tp > 1 and world != args.tp:
        raise SystemExit(f"--tp {args.tp} needs a world of {args.tp} ranks (got {world})")
    if os.environ.get("RB_WATCHDOG_S"):  # debug: every thread's Python stack to stderr, then exit
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["RB_WATCHDOG_S"]), exit=True)

    import torch

    from paper_2601_11822_b200.replicas import shard_items
    from paper_2601_11822_b200.specs import ARCHS
    from paper_2601_11822_b200.traffic import WorkloadSpec, synthesize

    torch.cuda.set_device(local)
    arch = ARCHS[args.model]
    peaks = _peaks()
    # trace long enough for warm-up + K steps (~20 ms per step at steady state) and >= 60 s so
    # the run-level rate is not dominated by the ramp
    duration = args.duration or max(60.0, 8.0 + (args.warmup + args.steps) * 0.02 * 1.6)
    horizon = int(duration * 1e6)
    tp = args.tp if args.tp > 1 else 1
    trace = synthesize(WorkloadSpec(qps=args.qps * (world // tp), duration_s=duration, seed=42,
                                    mean_prompt_tokens=PROMPT, mean_output_tokens=OUTPUT, sigma=0.0))
    channel = None
    tp_ex = None
    if tp > 1:
        import torch.distributed as dist

        from paper_2601_11822_b200.tp_engine import CommandChannel, attach_leader, serve_worker
        from paper_2601_11822_b200.tp_serve import build_tp_executor

        host = dist.new_group(backend="gloo")
        tp_ex = build_tp_executor(arch, rank, world, host, ar=args.tp_ar, device=f"cuda:{local}",
                                  static_decode_sms=args.decode_sms, max_batch=args.max_batch, chunk_tokens=2048,
                                  max_context=PROMPT + OUTPUT + 64, num_slots=4096,
                                  kv_memory_fraction=args.kv_memory_fraction, probe_attention=(rank == 0))
        channel = CommandChannel(host)
        if rank != 0:
            tp_ex.warmup()  # the same captures, in the same order, as rank 0's serve()
            n = serve_worker(tp_ex, channel)
            print(json.dumps({"tp_rank": rank, "commands": n, "frames": channel.frames}), file=sys.stderr)
            tp_ex.close()
            return
        attach_leader(tp_ex, channel)
        items = trace
    else:
        items = shard_items(trace, rank, world)

    if tp > 1:
        try:
            main_res = serve(args, tp_ex.arch, items, horizon, args.engine, 0, 1, local, primary=True, executor=tp_ex)
        finally:
            from paper_2601_11822_b200.tp_engine import stop_workers

            stop_workers(channel)
    else:
        main_res = serve(args, arch, items, horizon, args.engine, rank, world, local, primary=True)
    ex = main_res.pop("ex", None)
    part = main_res.pop("part", None)

    # isolated probe on the full device (secondary; the in-situ number is the roofline)
    iso = None
    if ex is not None:
        mB = int(round(main_res["mean_batch"] or 64))
        mctx = int(round(main_res["mean_ctx"] or PROMPT + OUTPUT // 2))
        full = ex._partitions[None]
        iso = time_decode_attention(ex.runner, full.ds, mB, mctx, full.d_sms)
        ex.close()
        del ex, part
    _free_cuda()

    comp = None
    if args.compare != "none":
        comp = serve(args, arch, items, horizon, args.compare, rank, world, local, primary=False)
        _free_cuda()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle.cpu_baseline import run_sample

        cpu = run_sample(arch, PROMPT, OUTPUT, batch=8, decode_steps=1, prefill_tokens=32)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank != 0:
        return

    def constrained(p):
        return p["tokens_per_s"] if p["itl_p99_us"] <= SLO_ITL_US else 0.0

    m = main_res
    pooled = m["pooled"]
    hbm = peaks["hbm_gbs"]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            nt = json.load(fh)["decode_attn_tc_kernel"]
        ratio = (nt["dram_bytes_read"] + nt["dram_bytes_write"]) / nt["algorithmic_bytes"]
    except (OSError, KeyError, ValueError):
        ratio = None
    pr = m["probe"]
    per_launch_bytes = pr["bytes"] / pr["launches"] if pr["launches"] else 0.0
    achieved = pr["bytes"] / pr["ms"] / 1e6 if pr["ms"] else None
    if ratio is not None and per_launch_bytes:
        traffic = ratio * per_launch_bytes
    steps = max(1, m["steps"])
    value = constrained(pooled)
    part = partition_bound(pr["by_sms"], (m["clocks"] or {}).get("sm_mhz"), hbm)
    line = {
        "metric": "SLO-constrained output tokens/s per GPU (p99 ITL<=SLO); p50 TTFT; p99 ITL",
        "value": value,
        "unit": "output tokens/s",
        "n_gpus": world,
        "steps": m["steps"],
        "warmup": args.warmup,
        "ms_per_step": m["ms"] / steps if m["complete"] else None,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": f"synthetic (random-init {args.model} weights of the real shapes, synthesize() trace)",
        "config": {
            "workload": (f"cfg3: {args.model} bf16, measured ARM ("
                         + (f"measured B200 tables, {args.arm_policy} policy" if m["policy"] else
                            "reference allocate()")
                         + f" at every launch; OVERALLOCATE -> both phases on {m['total_sms']} SMs, PARTITION -> "
                           f"green-context split)" if args.arm and args.engine == "rapid" else
                         f"{args.engine}: {args.model} bf16" if args.engine != "rapid" else
                         (f"cfg4: {args.model} bf16 TP={world} (rank 0 engine, workers replay its device "
                          f"commands), static split decode {args.decode_sms} SMs" if args.tp > 1 else
                          f"cfg2: {args.model} bf16, static split decode {args.decode_sms} SMs"))
                        + f", trace in {PROMPT}/out {OUTPUT} sigma=0 at {args.qps} QPS per replica for "
                          f"{duration:.0f} s, request i -> replica i mod {world}",
            "qps_per_replica": args.qps,
            "parallelism": f"tp{world} ({args.tp_ar} all-reduce)" if args.tp > 1 else f"replicas x{world}",
            "l2": "inputs > L2 (KV + weights ~30 GB per step); no flush",
            "step": "one decode iteration (CUDA-graph replay); prefill runs concurrently on its partition"
                    if args.engine == "rapid" else "one fused hybrid iteration (decode rows + one prefill chunk)",
            "engine": args.engine,
            "max_batch": args.max_batch,
        },
        "value_definition": ("reference summarize().tokens_per_s (metrics.py:146-200) over [10% horizon, horizon], "
                             "pooled over replicas (whole job); 0 when pooled p99 ITL > SLO"),
        "per_gpu": value / world,
        "tokens_per_s_unconstrained": pooled["tokens_per_s"],
        "p50_ttft_ms": pooled["ttft_p50_us"] / 1e3,
        "p99_itl_ms": pooled["itl_p99_us"] / 1e3,
        "p95_itl_ms": pooled["itl_p95_us"] / 1e3,
        "slo_itl_ms": SLO_ITL_US / 1e3,
        "slo_met": bool(pooled["itl_p99_us"] <= SLO_ITL_US),
        "goodput_req_s": pooled["goodput"],
        "per_replica_tokens_per_s": pooled["per_replica_tokens_per_s"],
        "device_window": {"tokens_per_s": m["tokens"] / (m["ms"] / 1e3) if m["complete"] else None,
                          "steps": m["steps"], "ms_per_step": m["ms"] / steps if m["complete"] else None,
                          "mean_decode_batch": m["mean_batch"], "mean_context": m["mean_ctx"],
                          "note": "output tokens of the K timed decode steps / their CUDA-event time (max over ranks)"},
        "e2e": {"value": m["tokens"] / m["host_s"] if m["complete"] else 0.0, "unit": "output tokens/s",
                "h2d_bytes_per_step": m["h2d"], "d2h_bytes_per_step": m["d2h"],
                "note": "host wall clock over the same K steps through RapidEngine/B200Executor (pinned H2D of "
                        "step inputs + block-table deltas + prefill ids, D2H of sampled ids, every step)"},
        "roofline": {"kernel": "decode_attn_tc_kernel (K3)", "bound": "hbm", "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm if achieved else None, "traffic": traffic,
                     "measured": (f"in situ: CUDA events around layer {arch.layers // 2}'s decode attention inside "
                                  f"the decode graphs, {pr['launches']} launches over the K timed steps on the ARM's "
                                  f"partitions; {per_launch_bytes:.0f} algorithmic B per launch on average"),
                     "by_decode_sms": {k: {"gbs": v["gbs"], "launches": v["launches"]}
                                       for k, v in pr["by_sms"].items()},
                     "partition_bound": part,
                     "traffic_src": "profiles/ncu_traffic.json (dram read+write / algorithmic bytes of one "
                                    "ncu --set full launch) x the mean in-situ launch bytes",
                     "isolated_full_device": (None if iso is None else
                                              {"sms": m["total_sms"], "gbs": iso["gbs"], "frac": iso["gbs"] / hbm,
                                               "B": iso["B"], "ctx": iso["ctx"], "us": round(iso["ms"] * 1e3, 1)}),
                     "peak_src": peaks["_src"]},
        "gpu_launches": m["launches"],
        "clocks": m["clocks"] or {"sm_mhz": None, "sm_max_mhz": None, "reasons": []},
        "tokens_per_joule": _tpj(m),
        "cpu_baseline": cpu,
        "run_wall_s": m["run_wall_s"],
        "arm_decisions": m["arm_decisions"],
        "stream_duty": m["duty"],
        "host_loop": {"decode_completion_to_next_launch": m["host_gap"], "poll_sleep_us": args.poll_sleep_us,
                      "us_per_step_by_stage": m["host_prof"]},
        "requests": m["requests"],
        "finished": m["finished_all"],
        "profiles": os.path.join(ROOT, "profiles"),
    }
    if comp is not None:
        cp = comp["pooled"]
        line["comparator"] = {
            "engine": comp["engine"], "value": constrained(cp), "tokens_per_s_unconstrained": cp["tokens_per_s"],
            "p99_itl_ms": cp["itl_p99_us"] / 1e3, "p50_ttft_ms": cp["ttft_p50_us"] / 1e3,
            "slo_met": bool(cp["itl_p99_us"] <= SLO_ITL_US), "goodput_req_s": cp["goodput"],
            "device_window_tokens_per_s": comp["tokens"] / (comp["ms"] / 1e3) if comp["complete"] else None,
            "mean_decode_batch": comp["mean_batch"], "run_wall_s": comp["run_wall_s"],
            "max_batch": args.compare_max_batch,
            "clocks": comp["clocks"],
            "stream_duty": comp["duty"]["decode"],
            "host_gap": comp["host_gap"],
            "tokens_per_joule": _tpj(comp),
            "note": "same trace, same engine code, same run; chunked-prefill hybrid batching on the whole device"}
        cv = constrained(cp)
        line["vs_comparator"] = value / cv if cv else None
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
