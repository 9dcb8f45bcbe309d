"""Generate the scheduler / ARM / block-accounting golden fixtures from the
reference simulator itself (arxiv/paper_2601_11822 `pdsim`).

Run HERE (the reference exists only in this container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.json. Tests read only these JSON files, so they also run
where /root/reference is absent. Every case pins bit-exact behaviour of the
reference: per-request records, pool occupancy series, busy intervals, ARM
decision sequences, and cost-model values.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("PDSIM_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import pdsim.engines.rapid as ref_rapid  # noqa: E402
from pdsim.config import load_gpu_spec, load_model_spec  # noqa: E402
from pdsim.core import GpuSpec, ModelSpec  # noqa: E402
from pdsim.costmodel import (  # noqa: E402
    CostParams,
    allocate,
    build_profile,
    decode_time,
    hybrid_time,
    overlapped_times,
    prefill_time,
    profile_lines,
)
from pdsim.core import AllocationDecision, AllocationMode, OVERALLOCATE  # noqa: E402
from pdsim.engines import build_engine  # noqa: E402
from pdsim.kvcache import BlockPool  # noqa: E402
from pdsim.metrics import SloSpec, summarize  # noqa: E402
from pdsim.runner import check_invariants  # noqa: E402
from pdsim.sim import Simulation  # noqa: E402
from pdsim.workload import WorkloadSpec, synthesize  # noqa: E402

B200 = GpuSpec("b200", 148, 1.381e15, 6.5434e12, 1.79e11, 10.0, 7.7e11)
# Llama-3.1-8B analytic spec (flops ~ 2 x params, bf16 weights)
LLAMA8B = ModelSpec("llama3.1-8b", 32, 8, 128, 2, 2 * 8.03e9, 2 * 8.03e9)
TINY = ModelSpec("tiny", 4, 2, 128, 2, 2 * 62.9e6, 2 * 62.9e6)


def digest(requests) -> str:
    h = hashlib.sha256()
    for r in sorted(requests, key=lambda r: r.id):
        h.update(repr((r.id, r.state.value, tuple(r.token_times_us), r.decode_participations, r.preemptions,
                       tuple((s.value, t) for s, t in r.history))).encode())
    return h.hexdigest()


def records(requests):
    return [
        dict(id=r.id, state=r.state.value, tokens=list(r.token_times_us), parts=r.decode_participations,
             pre=r.preemptions, hist=[[s.value, t] for s, t in r.history])
        for r in sorted(requests, key=lambda r: r.id)
    ]


def dec(d):
    return [d.mode.value, d.cu_fraction_prefill, d.cu_fraction_decode, d.slo_risk]


def run_case(label, model, gpu, tp, slo, spec=None, items=None, horizon=None, engine_params=None, pool_blocks=None,
             full=False):
    log = []
    orig = ref_rapid.allocate

    def spy(*a, **k):
        d = orig(*a, **k)
        log.append(dec(d))
        return d

    ref_rapid.allocate = spy
    try:
        engine = build_engine(label, model, gpu, tp, CostParams(), slo, engine_params or {})
        if pool_blocks is not None:
            engine.pool = BlockPool(pool_blocks, 16, name="gpu0")
            engine.pools = {"gpu0": engine.pool}
        if items is None:
            items = synthesize(spec)
            horizon = int(spec.duration_s * 1e6)
        sim = Simulation(until_us=horizon)
        engine.prime(sim, items)
        counts = {}
        inner = engine.on_event

        def handler(s, ev):
            counts[ev.kind.value] = counts.get(ev.kind.value, 0) + 1
            inner(s, ev)

        sim.run(handler)
        check_invariants(engine)
    finally:
        ref_rapid.allocate = orig
    summ = summarize(engine.label, spec.qps if spec else 0.0, engine.requests, slo, sim.horizon_us,
                     engine.busy_intervals, engine.pools)
    out = dict(
        label=label,
        n=len(engine.requests),
        digest=digest(engine.requests),
        events=counts,
        preemptions=sum(r.preemptions for r in engine.requests),
        finished=sum(1 for r in engine.requests if r.state.value == "finished"),
        summary={k: getattr(summ, k) for k in ("tokens_per_s", "requests_per_s", "goodput", "itl_goodput",
                                                "ttft_p95_us", "itl_p95_us", "compute_util", "mem_util")},
        pool_blocks=engine.pool.total_blocks,
        n_decisions=len(log),
        decisions_sha=hashlib.sha256(json.dumps(log).encode()).hexdigest(),
        partition_decisions=sum(1 for d in log if d[0] == "partition"),
    )
    if full:
        out["records"] = records(engine.requests)
        out["occupancy"] = [list(x) for x in engine.pool._occupancy]
        out["busy"] = [list(x) for x in engine.busy_intervals["gpu0"]]
        out["decisions"] = log
    return out


def main():
    mi300 = load_gpu_spec("mi300x-like")
    m70 = load_model_spec("llama70b-like")
    cases = {}
    # SURVEY.md Appendix A fixtures
    cases["F1"] = run_case("rapid", m70, mi300, 2, SloSpec(), WorkloadSpec(qps=5.0, duration_s=300.0, seed=42))
    cases["F2"] = run_case("rapid", m70, mi300, 2, SloSpec(itl_slo_us=50_000),
                           WorkloadSpec(qps=8.0, duration_s=120.0, seed=42, mean_prompt_tokens=2048,
                                        mean_output_tokens=1024, sigma=0.0))
    cases["F2_hybrid512"] = run_case("hybrid-512", m70, mi300, 2, SloSpec(itl_slo_us=50_000),
                                     WorkloadSpec(qps=8.0, duration_s=60.0, seed=42, mean_prompt_tokens=2048,
                                                  mean_output_tokens=1024, sigma=0.0))
    # cfg 1: tiny model, first 64 requests of the cfg-1 trace, full records
    spec1 = WorkloadSpec(qps=4.0, duration_s=30.0, seed=0, mean_prompt_tokens=64, mean_output_tokens=16)
    items1 = synthesize(spec1)[:64]
    slo = SloSpec(itl_slo_us=50_000)
    cases["tiny_rapid_2048"] = run_case("rapid", TINY, B200, 1, slo, items=items1, full=True)
    cases["tiny_rapid_32"] = run_case("rapid", TINY, B200, 1, slo, items=items1, engine_params={"chunk_tokens": 32},
                                      full=True)
    cases["tiny_rapid_pool64"] = run_case("rapid", TINY, B200, 1, slo, items=items1,
                                          engine_params={"chunk_tokens": 32}, pool_blocks=64, full=True)
    cases["tiny_hybrid_64_pool64"] = run_case("hybrid-64", TINY, B200, 1, slo, items=items1, pool_blocks=64,
                                              full=True)
    cases["tiny_rapid_horizon"] = run_case("rapid", TINY, B200, 1, slo, items=items1, horizon=8_000_000,
                                           pool_blocks=40, full=True)
    # cfg 2/3 shape on B200 (8B, 1024/256 fixed lengths), 30 s at 48 QPS
    spec2 = WorkloadSpec(qps=48.0, duration_s=30.0, seed=42, mean_prompt_tokens=1024, mean_output_tokens=256,
                         sigma=0.0)
    cases["b200_8b_rapid"] = run_case("rapid", LLAMA8B, B200, 1, slo, spec2)
    cases["b200_8b_hybrid512"] = run_case("hybrid-512", LLAMA8B, B200, 1, slo, spec2)
    with open(os.path.join(HERE, "engines.json"), "w") as fh:
        json.dump(cases, fh, indent=None, separators=(",", ":"))

    # ---------------- cost model / ARM known answers
    p = CostParams()
    kat = {"prefill": [], "decode": [], "overlapped": [], "hybrid": [], "allocate": [], "profiles": {}}
    for model_name, model, gpu in (("70b_mi300_tp2", m70, mi300.aggregate(2)), ("8b_b200", LLAMA8B, B200),
                                   ("tiny_b200", TINY, B200)):
        for tok in (1, 17, 512, 1024, 2048, 8192):
            for cu in (1 / 148, 0.25, 0.4, 0.5, 0.73, 1.0):
                for conc in (False, True):
                    kat["prefill"].append([model_name, tok, cu, conc, prefill_time(tok, cu, model, gpu, p, conc)])
        for b in (1, 7, 64, 256):
            for kv in (0, 1000, 300_000):
                for cu in (1 / 304, 0.1, 0.4, 1.0):
                    for conc in (False, True):
                        kat["decode"].append([model_name, b, kv, cu, conc,
                                              decode_time(b, kv, cu, model, gpu, p, conc)])
        for pt in (0, 1, 2048):
            for b in (0, 1, 160):
                for mode in ("over", "part"):
                    alloc = OVERALLOCATE if mode == "over" else AllocationDecision(AllocationMode.PARTITION, 0.6,
                                                                                 0.4)
                    kat["overlapped"].append([model_name, pt, b, 1000 * b, mode,
                                              list(overlapped_times(pt, b, 1000 * b, alloc, model, gpu, p))])
        for pt in (0, 5, 512):
            for b in (0, 3, 256):
                if pt or b:
                    kat["hybrid"].append([model_name, pt, b, 777 * b, hybrid_time(pt, b, 777 * b, model, gpu, p)])
        for slo_us in (10_000, 20_000, 50_000, 100_000):
            prof = build_profile(model, gpu, p, slo_us)
            kat["profiles"][f"{model_name}@{slo_us}"] = profile_lines(prof)
            for b in (0, 1, 33, 64, 160, 256, 300):
                for pt in (0, 128, 2048):
                    kat["allocate"].append([model_name, slo_us, b, pt, dec(allocate(prof, b, pt, slo_us, model, gpu,
                                                                                    p))])
    with open(os.path.join(HERE, "costmodel.json"), "w") as fh:
        json.dump(kat, fh, indent=None, separators=(",", ":"))

    # ---------------- workload generator known answers
    wl = {}
    for name, spec in {
        "cfg1": spec1,
        "cfg2": WorkloadSpec(qps=32.0, duration_s=120.0, seed=42, mean_prompt_tokens=1024, mean_output_tokens=256,
                             sigma=0.0),
        "default": WorkloadSpec(qps=5.0, duration_s=60.0, seed=7),
        "cfg5": WorkloadSpec(qps=6.0, duration_s=60.0, seed=42, mean_prompt_tokens=8192, mean_output_tokens=128,
                             sigma=0.0),
    }.items():
        items = synthesize(spec)
        wl[name] = dict(spec=[spec.qps, spec.duration_s, spec.seed, spec.mean_prompt_tokens, spec.mean_output_tokens,
                              spec.sigma], n=len(items),
                        sha=hashlib.sha256(repr([(i.arrival_us, i.prompt_tokens, i.output_tokens)
                                                 for i in items]).encode()).hexdigest(),
                        head=[[i.arrival_us, i.prompt_tokens, i.output_tokens] for i in items[:20]])
    with open(os.path.join(HERE, "workload.json"), "w") as fh:
        json.dump(wl, fh, indent=None, separators=(",", ":"))
    print({k: (v["n"], v["preemptions"], v["partition_decisions"]) for k, v in cases.items()})


if __name__ == "__main__":
    main()
