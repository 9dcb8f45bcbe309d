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
