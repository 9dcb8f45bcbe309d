"""Trace-replay parity of GPU runs (north star "scheduler admission /
ordering bit-exact").

A real-time RAPID run on the B200 records, per launch, the event time that kicked it and
the time its completion was observed (RapidEngine(record_launches=True)). Replaying that
timeline on the virtual clock — every launch priced at its recorded duration, no host gap
(cpu_us = 0) — must reproduce the GPU run's scheduling exactly: the same per-request
records (history, token stamps, participations, preemptions: the Appendix-A digest), the
same ARM decision sequence and the same pool occupancy series.

  * GPU test: record a run, replay it through this package's engine, compare; the trace is
    also written to gpurun_out/replay/ (the committed fixtures under tests/golden/ come from
    there).
  * CPU test: replay every committed fixture through this package's engine AND through the
    reference pdsim RapidEngine itself (pkg/src/pdsim/engines/rapid.py:148-323, pricing
    monkeypatched at its call sites :171-189 / :266-293, allocate() left as is), and
    compare both with the GPU run's recorded digest / decisions / occupancy.
"""

from __future__ import annotations

import glob
import hashlib
import json
import os
import sys
from collections import deque

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"


def _sha(obj) -> str:
    return hashlib.sha256(json.dumps(obj).encode()).hexdigest()


def _specs(fx):
    from paper_2601_11822_b200.arm import CostParams
    from paper_2601_11822_b200.slo import SloSpec
    from paper_2601_11822_b200.specs import GpuSpec, ModelSpec

    return ModelSpec(**fx["model"]), GpuSpec(**fx["gpu"]), CostParams(), SloSpec(itl_slo_us=fx["slo_us"])


def _items(fx):
    from paper_2601_11822_b200.traffic import WorkloadItem

    return [WorkloadItem(*it) for it in fx["items"]]


def _check_ours(fx):
    from paper_2601_11822_b200.harness import decision_tuples, replay_rapid
    from paper_2601_11822_b200.lifecycle import request_digest

    model, gpu, params, slo = _specs(fx)
    eng = replay_rapid(_items(fx), [tuple(x) for x in fx["launch_log"]], model, gpu, params, slo,
                       chunk_tokens=fx["chunk_tokens"], max_batch=fx["max_batch"], num_blocks=fx["num_blocks"],
                       horizon_us=fx["horizon_us"])
    assert request_digest(eng.requests) == fx["digest"]
    assert _sha([list(d) for d in decision_tuples(eng.decision_log)]) == fx["decisions_sha"]
    assert _sha(eng.pool.occupancy_series) == fx["occupancy_sha"]
    return eng


def reference_replay(fx):
    """The unmodified reference RapidEngine on the recorded timeline."""
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import pdsim.engines.rapid as R
    from pdsim.core import GpuSpec, ModelSpec
    from pdsim.costmodel import CostParams
    from pdsim.kvcache import BlockPool
    from pdsim.metrics import SloSpec
    from pdsim.sim import Simulation
    from pdsim.workload import WorkloadItem

    durs = {"prefill": deque(), "decode": deque()}
    for phase, start, end in fx["launch_log"]:
        durs[phase].append(end - start)
    eng = R.RapidEngine(ModelSpec(**fx["model"]), GpuSpec(**fx["gpu"]), CostParams(),
                        SloSpec(itl_slo_us=fx["slo_us"]), chunk_tokens=fx["chunk_tokens"], max_batch=fx["max_batch"])
    eng.cpu_us = 0
    eng.pool = BlockPool(fx["num_blocks"], 16, name="gpu0")
    eng.pools = {"gpu0": eng.pool}
    phase = [None]
    decisions = []
    orig = {k: getattr(R, k) for k in ("allocate", "prefill_time", "decode_time", "overlapped_times")}

    def allocate(*a, **k):
        d = orig["allocate"](*a, **k)
        decisions.append([phase[0], d.mode.value, d.cu_fraction_prefill, d.cu_fraction_decode, d.slo_risk])
        return d

    def price(*a, **k):
        return durs[phase[0]].popleft()

    def overlapped(*a, **k):
        v = durs[phase[0]].popleft()
        return v, v

    p_kick, d_kick = eng._p_kick, eng._d_kick

    def pk(sim):
        phase[0] = "prefill"
        p_kick(sim)

    def dk(sim):
        phase[0] = "decode"
        d_kick(sim)

    eng._p_kick, eng._d_kick = pk, dk
    try:
        R.allocate, R.prefill_time, R.decode_time, R.overlapped_times = allocate, price, price, overlapped
        sim = Simulation(until_us=fx["horizon_us"])
        eng.prime(sim, [WorkloadItem(*it) for it in fx["items"]])
        sim.run(eng.on_event)
    finally:
        for k, v in orig.items():
            setattr(R, k, v)
    assert not durs["prefill"] and not durs["decode"], "reference replay made fewer launches than the GPU run"
    return eng, decisions


def _fixtures():
    return sorted(glob.glob(os.path.join(GOLDEN, "replay_*.json")))


@pytest.mark.parametrize("path", _fixtures(), ids=lambda p: os.path.basename(p))
def test_replay_committed_gpu_trace(path):
    with open(path) as fh:
        fx = json.load(fh)
    eng = _check_ours(fx)
    assert sum(r.state.value == "finished" for r in eng.requests) == fx["finished"]
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not mounted: replayed through this package's engine only")
    from paper_2601_11822_b200.lifecycle import request_digest

    ref, decisions = reference_replay(fx)
    assert request_digest(ref.requests) == fx["digest"], "reference scheduling differs from the GPU run"
    assert _sha(decisions) == fx["decisions_sha"]
    assert _sha(ref.pool._occupancy) == fx["occupancy_sha"]


def test_fixtures_present():
    assert _fixtures(), "no recorded GPU trace under tests/golden/replay_*.json"


@pytest.mark.gpu
@pytest.mark.parametrize("name,compress,chunk,slo_us,num_blocks",
                         [("cfg1_x1000_chunk32_slo60us", 1000, 32, 60, 1024),
                          ("cfg1_x200_pool64_chunk32", 200, 32, 50_000, 64),
                          ("cfg1_x1000_chunk2048_slo60us", 1000, 2048, 60, 1024)])
def test_record_and_replay_gpu(name, compress, chunk, slo_us, num_blocks):
    """Serve the cfg-1 trace (time-compressed so batches form) on the B200 with the reference
    ARM (allocate(); a 60 us SLO makes it PARTITION whenever both phases have work, so launches move between
    green-context splits), record the timeline, replay it, compare."""
    from oracle.llama_fp32 import init_state
    from paper_2601_11822_b200.arm import CostParams
    from paper_2601_11822_b200.engines.rapid import RapidEngine
    from paper_2601_11822_b200.executor_b200 import B200Executor
    from paper_2601_11822_b200.harness import decision_tuples, run_items
    from paper_2601_11822_b200.lifecycle import request_digest
    from paper_2601_11822_b200.model import DecoderWeights
    from paper_2601_11822_b200.slo import SloSpec
    from paper_2601_11822_b200.specs import ARCHS, b200_spec
    from paper_2601_11822_b200.traffic import WorkloadItem, WorkloadSpec, synthesize

    arch = ARCHS["tiny"]
    items = [WorkloadItem(it.arrival_us // compress, it.prompt_tokens, it.output_tokens)
             for it in synthesize(WorkloadSpec(qps=4.0, duration_s=30.0, seed=0, mean_prompt_tokens=64,
                                               mean_output_tokens=16))[:64]]
    ex = B200Executor(arch, weights=DecoderWeights.from_state(arch, init_state(arch, seed=0)), max_batch=32,
                      chunk_tokens=chunk, num_blocks=num_blocks, max_context=1024, num_slots=128)
    ex.warmup()
    model, gpu, params, slo = arch.model_spec(), b200_spec(), CostParams(), SloSpec(itl_slo_us=slo_us)
    res = run_items("rapid", items, model, gpu, params, slo,
                    engine_factory=lambda: RapidEngine(model, gpu, params, slo, chunk_tokens=chunk, max_batch=32,
                                                       executor=ex, record_decisions=True, record_launches=True))
    eng = res.engine
    fx = {
        "name": name, "model": dict(vars(model)), "gpu": dict(vars(gpu)), "slo_us": slo_us, "chunk_tokens": chunk,
        "max_batch": 32, "num_blocks": num_blocks, "horizon_us": None,
        "items": [[it.arrival_us, it.prompt_tokens, it.output_tokens] for it in items],
        "launch_log": [list(x) for x in eng.launch_log],
        "digest": request_digest(eng.requests),
        "decisions_sha": _sha([list(d) for d in decision_tuples(eng.decision_log)]),
        "occupancy_sha": _sha(eng.pool.occupancy_series),
        "finished": sum(r.state.value == "finished" for r in eng.requests),
        "preemptions": sum(r.preemptions for r in eng.requests),
        "partition_decisions": sum(1 for _, d in eng.decision_log if d.mode.value == "partition"),
        "decisions": len(eng.decision_log),
    }
    os.makedirs(os.path.join(ROOT, "gpurun_out", "replay"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "replay", f"replay_{name}.json"), "w") as fh:
        json.dump(fx, fh)
    print(name, {k: fx[k] for k in ("finished", "preemptions", "partition_decisions", "decisions")},
          len(fx["launch_log"]), "launches")
    _check_ours(fx)
    if num_blocks == 64:
        assert fx["preemptions"] >= 1
    if slo_us == 60:
        assert 0 < fx["partition_decisions"] < fx["decisions"], "want both OVERALLOCATE and PARTITION launches"
    ex.close()
