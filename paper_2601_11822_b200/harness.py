"""Driving one run and checking its end state.

`check_invariants` is the reference's post-run checker (pkg/src/pdsim/
runner.py:45-69): pools drained, every request terminal, finished requests
delivered exactly their output, preemption back-edges == preemption count,
monotone history. `run_one` mirrors runner.run_one (:72-97) for an
items list; with a GPU executor it runs under `RealTimeLoop`.
"""

from __future__ import annotations

from dataclasses import dataclass

from paper_2601_11822_b200.clock import RealTimeLoop, Simulation
from paper_2601_11822_b200.engines import EngineBase, build_engine
from paper_2601_11822_b200.lifecycle import RequestState
from paper_2601_11822_b200.slo import RequestRow, Summary, evaluate_request, summarize


def check_invariants(engine: EngineBase) -> None:
    problems: list[str] = []
    for name, pool in engine.pools.items():
        if pool.used_blocks != 0:
            problems.append(f"pool {name} still holds {pool.used_blocks} blocks")
    for r in engine.requests:
        if r.state not in (RequestState.FINISHED, RequestState.REJECTED):
            problems.append(f"request {r.id} ended non-terminal in {r.state.value}")
        if r.state is RequestState.FINISHED and r.delivered_tokens != r.output_tokens:
            problems.append(f"request {r.id} finished with {r.delivered_tokens}/{r.output_tokens} tokens")
        h = r.history
        back = sum(1 for (a, _), (b, _) in zip(h, h[1:])
                   if a is RequestState.DECODING and b is RequestState.PENDING_KV)
        if back != r.preemptions:
            problems.append(f"request {r.id} preemption count mismatch")
        if any(t1 > t2 for (_, t1), (_, t2) in zip(h, h[1:])):
            problems.append(f"request {r.id} history times not monotone")
    if problems:
        raise RuntimeError("post-run invariant violations: " + "; ".join(problems[:5]))


@dataclass
class RunResult:
    summary: Summary
    rows: list[RequestRow]
    engine: EngineBase
    horizon_us: int


def run_items(label: str, items, model, gpu, params, slo, *, tp: int = 1, engine_params: dict | None = None,
              executor=None, horizon_us: int | None = None, qps: float = 0.0, realtime: bool | None = None,
              engine_factory=None) -> RunResult:
    """Run one engine over `items` and summarise (runner.run_one semantics)."""
    if engine_factory is not None:
        engine = engine_factory()
    else:
        engine = build_engine(label, model, gpu, tp, params, slo, engine_params, executor=executor)
    rt = getattr(engine.executor, "realtime", False) if realtime is None else realtime
    sim = RealTimeLoop(until_us=horizon_us) if rt else Simulation(until_us=horizon_us)
    engine.prime(sim, items)
    sim.run(engine.on_event)
    check_invariants(engine)
    rows = [evaluate_request(r, slo) for r in engine.requests]
    summary = summarize(engine.label, qps, engine.requests, slo, sim.horizon_us, engine.busy_intervals, engine.pools)
    return RunResult(summary, rows, engine, sim.horizon_us)


def decision_tuples(decision_log) -> list[tuple]:
    return [(ph, d.mode.value, d.cu_fraction_prefill, d.cu_fraction_decode, d.slo_risk) for ph, d in decision_log]


def replay_rapid(items, launch_log, model, gpu, params, slo, *, chunk_tokens: int, max_batch: int,
                 num_blocks: int | None, horizon_us: int | None = None):
    """Trace replay: re-run RAPID on the virtual clock with every launch
    priced at the duration a GPU run recorded for it (executor.ReplayExecutor) and no host
    gap (cpu_us = 0: the real-time engine's launches start at the event that kicked them).
    Returns the engine; its requests / decision_log / pool occupancy are then comparable
    with the GPU run's."""
    from paper_2601_11822_b200.engines.rapid import RapidEngine
    from paper_2601_11822_b200.executor import ReplayExecutor

    ex = ReplayExecutor(launch_log, num_blocks)
    eng = RapidEngine(model, gpu, params, slo, chunk_tokens=chunk_tokens, max_batch=max_batch, executor=ex,
                      record_decisions=True, record_launches=True)
    eng.cpu_us = 0
    sim = Simulation(until_us=horizon_us)
    eng.prime(sim, items)
    sim.run(eng.on_event)
    check_invariants(eng)
    if not ex.exhausted():
        raise RuntimeError("replay diverged: the GPU run recorded launches the replay never made")
    return eng
