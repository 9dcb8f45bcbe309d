"""Paged block manager: reference block counts under random traffic, the
physical-ID policy of SURVEY.md Appendix C.2 (pinned by this repo's goldens),
the device-table listener stream, and the replica (N>1) host path over gloo."""

import os
import random

import pytest

from paper_2601_11822_b200.blockpool import BlockPool, InsufficientCapacity
from paper_2601_11822_b200.replicas import ReplicaStats, reduce_stats, shard_items


class Recorder:
    def __init__(self):
        self.events = []

    def on_pages(self, rid, first, ids):
        self.events.append(("pages", rid, first, list(ids)))

    def on_release(self, rid):
        self.events.append(("release", rid))


def test_id_policy_golden():
    p = BlockPool(8, 16)
    rec = Recorder()
    p.listener = rec
    p.allocate(1, 33, 0)          # 3 pages
    p.allocate(2, 16, 1)          # 1 page
    assert p.block_ids(1) == [0, 1, 2] and p.block_ids(2) == [3]
    assert p.extend_to(2, 17, 2) == 1 and p.block_ids(2) == [3, 4]
    assert p.extend_to(2, 20, 3) == 0  # grow-only, already covered
    assert p.release(1, 4) == 3 and p.release(1, 4) == 0  # idempotent
    p.allocate(3, 40, 5)  # LIFO reuse in the original order: 0, 1, 2
    assert p.block_ids(3) == [0, 1, 2]
    with pytest.raises(InsufficientCapacity):
        p.allocate(4, 16 * 4, 6)  # 3 free, need 4 -> all or nothing
    assert p.free_blocks == 3 and not p.holds(4)
    assert rec.events == [("pages", 1, 0, [0, 1, 2]), ("pages", 2, 0, [3]), ("pages", 2, 1, [4]), ("release", 1),
                          ("pages", 3, 0, [0, 1, 2])]
    assert p.occupancy_series == [(0, 3), (1, 4), (2, 5), (4, 2), (5, 5)]


def test_ids_are_disjoint_and_counts_match_a_counts_only_model():
    """Random traffic: physical IDs never double-booked; counts equal the
    reference's counts-only semantics (kvcache.py:85-127), restated here."""
    rng = random.Random(7)
    p = BlockPool(97, 16)
    held: dict[int, int] = {}  # counts-only model
    used = 0
    t = 0
    for step in range(4000):
        t += rng.randint(0, 2)
        op = rng.random()
        rid = rng.randint(0, 40)
        if op < 0.4:
            tokens = rng.randint(1, 200)
            need = -(-tokens // 16)
            if rid in held:
                with pytest.raises(ValueError):
                    p.allocate(rid, tokens, t)
            elif need > 97 - used:
                with pytest.raises(InsufficientCapacity):
                    p.allocate(rid, tokens, t)
            else:
                p.allocate(rid, tokens, t)
                held[rid] = need
                used += need
        elif op < 0.7:
            if rid not in held:
                with pytest.raises(ValueError):
                    p.extend_to(rid, 10, t)
                continue
            tokens = rng.randint(1, 400)
            need = -(-tokens // 16)
            extra = max(0, need - held[rid])
            if extra > 97 - used:
                with pytest.raises(InsufficientCapacity):
                    p.extend_to(rid, tokens, t)
            else:
                assert p.extend_to(rid, tokens, t) == extra
                held[rid] += extra
                used += extra
        else:
            got = p.release(rid, t)
            assert got == held.pop(rid, 0)
            used -= got
        assert p.used_blocks == used and p.free_blocks == 97 - used
        ids = [i for r in held for i in p.block_ids(r)]
        assert len(ids) == len(set(ids)) == used
        assert all(0 <= i < 97 for i in ids)


def test_reference_blockpool_counts_if_available():
    """Live cross-check against the reference BlockPool when it is mounted."""
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not mounted")
    import sys

    sys.path.insert(0, src)
    from pdsim.kvcache import BlockPool as RefPool
    from pdsim.kvcache import InsufficientCapacity as RefIC

    rng = random.Random(11)
    a, b = BlockPool(50, 16), RefPool(50, 16)
    t = 0
    for _ in range(3000):
        t += rng.randint(0, 3)
        rid = rng.randint(0, 20)
        tok = rng.randint(1, 300)
        op = rng.choice(["alloc", "ext", "rel"])
        ra = rb = None
        for pool, ic in ((a, InsufficientCapacity), (b, RefIC)):
            try:
                r = getattr(pool, {"alloc": "allocate", "ext": "extend_to", "rel": "release"}[op])(
                    rid, *((tok, t) if op != "rel" else (t,)))
                res = ("ok", r)
            except ic:
                res = ("cap",)
            except ValueError:
                res = ("val",)
            if pool is a:
                ra = res
            else:
                rb = res
        assert ra == rb
        assert a.used_blocks == b.used_blocks
        assert a.occupancy_series == b._occupancy
    assert a.utilization(0, t + 1) == b.utilization(0, t + 1)


def test_shard_items_round_robin():
    items = list(range(10))
    shards = [shard_items(items, r, 3) for r in range(3)]
    assert shards == [[0, 3, 6, 9], [1, 4, 7], [2, 5, 8]]
    assert sorted(sum(shards, [])) == items


def _replica_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2601_11822_b200.arm import CostParams
    from paper_2601_11822_b200.harness import run_items
    from paper_2601_11822_b200.slo import SloSpec
    from paper_2601_11822_b200.specs import ARCHS, b200_spec
    from paper_2601_11822_b200.traffic import WorkloadSpec, synthesize

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    items = synthesize(WorkloadSpec(qps=20.0, duration_s=6.0, seed=3, mean_prompt_tokens=256, mean_output_tokens=32))
    mine = shard_items(items, rank, world)
    model = ARCHS["tiny"].model_spec()
    res = run_items("rapid", mine, model, b200_spec(), CostParams(), SloSpec(itl_slo_us=50_000),
                    horizon_us=6_000_000)
    toks = sum(len(r.token_times_us) for r in res.engine.requests)
    fin = sum(1 for r in res.engine.requests if r.state.value == "finished")
    agg = reduce_stats(ReplicaStats(toks, 6.0, fin, res.summary.itl_p99_us, res.summary.ttft_p50_us))
    from paper_2601_11822_b200.replicas import local_window_stats, pool_window_stats

    local = local_window_stats(res.engine.requests, SloSpec(itl_slo_us=50_000), 6_000_000)
    pooled = pool_window_stats(local)  # what bench.py reports at N > 1
    q.put((rank, toks, fin, agg, local, pooled))
    dist.destroy_process_group()


def test_replicas_gloo_world2():
    """world_size-2 gloo run of the replica path: each rank serves its shard
    with its own engine; the reduced totals equal the per-rank sums."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    tot = sum(o[1] for o in out)
    fin = sum(o[2] for o in out)
    for _, _, _, agg, _, _ in out:
        assert agg["tokens"] == tot and agg["finished"] == fin
        assert agg["window_s"] == 6.0
    # bench's pooled run-level stats: whole-job tokens / the common window, and the p99 ITL /
    # p50 TTFT over the UNION of both replicas' samples (not a max of per-rank percentiles)
    from paper_2601_11822_b200.slo import percentile_nearest_rank

    locs = [o[4] for o in out]
    gaps = [g for l in locs for g in l["gaps"]]
    ttfts = [t for l in locs for t in l["ttfts"]]
    for o in out:
        pooled = o[5]
        assert pooled["replicas"] == 2
        assert pooled["tokens_per_s"] == sum(l["stamps"] for l in locs) / locs[0]["window_s"]
        assert pooled["itl_p99_us"] == percentile_nearest_rank(gaps, 99.0)
        assert pooled["ttft_p50_us"] == percentile_nearest_rank(ttfts, 50.0)
