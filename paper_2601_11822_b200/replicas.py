"""Multi-GPU use where the path shards: one independent RAPID replica per GPU.

SURVEY.md §8(e): for 8B / 14B the work shards naturally by request —
request i goes to replica i mod N (the reference's own round-robin placement,
pkg/src/pdsim/engines/disagg.py:81-83). Replicas share nothing (own BlockPool,
green contexts, KV cache); there is no data-path collective. The only
cross-rank traffic is the end-of-run reduction of the metrics, done here over
torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass


def shard_items(items: list, rank: int, world: int) -> list:
    """Round-robin request placement, arrival order preserved within a replica."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return [it for i, it in enumerate(items) if i % world == rank]


@dataclass(frozen=True)
class ReplicaStats:
    tokens: float          # output tokens delivered in the measured window
    window_s: float        # window length (device time) on this replica
    finished: float
    itl_p99_us: float
    ttft_p50_us: float


def reduce_stats(local: ReplicaStats, group=None, device=None) -> dict:
    """Whole-job aggregate: tokens summed, window = max over ranks (the slowest
    replica bounds the job), latency percentiles = max over ranks (conservative)."""
    import torch
    import torch.distributed as dist

    v = torch.tensor([local.tokens, local.finished], dtype=torch.float64, device=device)
    m = torch.tensor([local.window_s, local.itl_p99_us, local.ttft_p50_us], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    tokens, finished = float(v[0]), float(v[1])
    window, itl, ttft = float(m[0]), float(m[1]), float(m[2])
    return {"tokens": tokens, "finished": finished, "window_s": window, "tokens_per_s": tokens / window if window > 0
            else 0.0, "itl_p99_us": itl, "ttft_p50_us": ttft}


def local_window_stats(requests, slo, horizon_us: int) -> dict:
    """The per-replica ingredients of summarize() (slo.py, reference metrics.py:146-200)
    that pool across replicas: in-window token stamps, finished-in-window counts, ITL gaps
    and TTFTs of finished in-window requests."""
    from paper_2601_11822_b200.slo import WARMUP_FRACTION, evaluate_request, itl_samples_us
    from paper_2601_11822_b200.lifecycle import RequestState

    cut = int(horizon_us * WARMUP_FRACTION)
    finished = [r for r in requests if r.arrival_us >= cut and r.state is RequestState.FINISHED]
    rows = [evaluate_request(r, slo) for r in finished]
    return {
        "stamps": sum(1 for r in requests for t in r.token_times_us if cut <= t <= horizon_us),
        "finished": len(finished),
        "ok_both": sum(1 for x in rows if x.meets_itl and x.meets_ttft),
        "gaps": [g for r in finished for g in itl_samples_us(r)],
        "ttfts": [x.ttft_us for x in rows if x.ttft_us >= 0],
        "window_s": (horizon_us - cut) / 1e6,
    }


def pool_window_stats(local: dict, group=None, pool: bool = True) -> dict:
    """Whole-job run-level metrics over all replicas: tokens/s = all in-window stamps / the
    (common) window, p99 ITL / p50 TTFT nearest-rank over the POOLED samples of every replica
    (not a max of per-rank percentiles). Every rank gets the result."""
    import torch.distributed as dist

    from paper_2601_11822_b200.slo import percentile_nearest_rank

    parts = [local]
    # pool=False: this rank's engine is the whole job (rank 0 of a TP group)
    if pool and dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        parts = [None] * dist.get_world_size(group)
        dist.all_gather_object(parts, local, group=group)
    window = max(p["window_s"] for p in parts)
    gaps = [g for p in parts for g in p["gaps"]]
    ttfts = [t for p in parts for t in p["ttfts"]]
    return {
        "replicas": len(parts),
        "tokens_per_s": sum(p["stamps"] for p in parts) / window,
        "per_replica_tokens_per_s": [p["stamps"] / p["window_s"] for p in parts],
        "goodput": sum(p["ok_both"] for p in parts) / window,
        "finished": sum(p["finished"] for p in parts),
        "itl_p99_us": percentile_nearest_rank(gaps, 99.0) if gaps else 0.0,
        "itl_p95_us": percentile_nearest_rank(gaps, 95.0) if gaps else 0.0,
        "ttft_p50_us": percentile_nearest_rank(ttfts, 50.0) if ttfts else -1.0,
        "window_s": window,
    }
