"""Bit-exact parity of the host engines / ARM / block accounting with the
reference simulator, through golden fixtures made by tests/golden/make_golden.py
(which imports the reference itself). CPU only."""

import hashlib
import json
import os

import pytest

from paper_2601_11822_b200.arm import (
    CostParams,
    allocate,
    build_profile,
    decode_time,
    hybrid_time,
    overlapped_times,
    prefill_time,
    profile_lines,
)
from paper_2601_11822_b200.blockpool import BlockPool
from paper_2601_11822_b200.clock import Simulation
from paper_2601_11822_b200.engines import build_engine
from paper_2601_11822_b200.harness import check_invariants
from paper_2601_11822_b200.lifecycle import request_digest
from paper_2601_11822_b200.slo import SloSpec, summarize
from paper_2601_11822_b200.specs import (
    LLAMA70B_LIKE,
    MI300X_LIKE,
    OVERALLOCATE,
    AllocationDecision,
    AllocationMode,
    GpuSpec,
    ModelSpec,
)
from paper_2601_11822_b200.traffic import WorkloadSpec, synthesize

GOLD = os.path.join(os.path.dirname(__file__), "golden")
B200 = GpuSpec("b200", 148, 1.381e15, 6.5434e12, 1.79e11, 10.0, 7.7e11)
LLAMA8B = ModelSpec("llama3.1-8b", 32, 8, 128, 2, 2 * 8.03e9, 2 * 8.03e9)
TINY = ModelSpec("tiny", 4, 2, 128, 2, 2 * 62.9e6, 2 * 62.9e6)
MODELS = {"70b_mi300_tp2": (LLAMA70B_LIKE, MI300X_LIKE.aggregate(2)), "8b_b200": (LLAMA8B, B200),
          "tiny_b200": (TINY, B200)}


@pytest.fixture(scope="module")
def engines_gold():
    with open(os.path.join(GOLD, "engines.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def cost_gold():
    with open(os.path.join(GOLD, "costmodel.json")) as fh:
        return json.load(fh)


def _dec(d):
    return [d.mode.value, d.cu_fraction_prefill, d.cu_fraction_decode, d.slo_risk]


def run_case(label, model, gpu, tp, slo, spec=None, items=None, horizon=None, engine_params=None, pool_blocks=None):
    engine = build_engine(label, model, gpu, tp, CostParams(), slo, engine_params or {})
    if hasattr(engine, "decision_log"):
        engine.decision_log = []
    if pool_blocks is not None:
        engine.pool = BlockPool(pool_blocks, 16, name="gpu0")
        engine.pools = {"gpu0": engine.pool}
    if items is None:
        items = synthesize(spec)
        horizon = int(spec.duration_s * 1e6)
    sim = Simulation(until_us=horizon)
    engine.prime(sim, items)
    counts = {}

    def handler(s, ev):
        counts[ev.kind.value] = counts.get(ev.kind.value, 0) + 1
        engine.on_event(s, ev)

    sim.run(handler)
    check_invariants(engine)
    summ = summarize(engine.label, spec.qps if spec else 0.0, engine.requests, slo, sim.horizon_us,
                     engine.busy_intervals, engine.pools)
    log = [_dec(d) for _, d in (getattr(engine, "decision_log", None) or [])]
    return engine, counts, summ, log


def _check(engine, counts, summ, log, gold, full=False):
    assert len(engine.requests) == gold["n"]
    assert counts == gold["events"]
    assert sum(r.preemptions for r in engine.requests) == gold["preemptions"]
    assert engine.pool.total_blocks == gold["pool_blocks"]
    for k, v in gold["summary"].items():
        assert getattr(summ, k) == v, k
    if engine.label == "rapid":
        assert len(log) == gold["n_decisions"]
        assert hashlib.sha256(json.dumps(log).encode()).hexdigest() == gold["decisions_sha"]
    assert request_digest(engine.requests) == gold["digest"]
    if full:
        recs = [dict(id=r.id, state=r.state.value, tokens=list(r.token_times_us), parts=r.decode_participations,
                     pre=r.preemptions, hist=[[s.value, t] for s, t in r.history])
                for r in sorted(engine.requests, key=lambda r: r.id)]
        assert recs == gold["records"]
        assert [list(x) for x in engine.pool.occupancy_series] == gold["occupancy"]
        assert [list(x) for x in engine.busy_intervals["gpu0"]] == gold["busy"]


def test_F1_overallocate_trace(engines_gold):
    """1,484 requests, all OVERALLOCATE."""
    g = engines_gold["F1"]
    out = run_case("rapid", LLAMA70B_LIKE, MI300X_LIKE, 2, SloSpec(), WorkloadSpec(qps=5.0, duration_s=300.0, seed=42))
    _check(*out, g)
    assert g["digest"] == "efd23e69a3ad022def88238176fddf6b885a7d517cd2ccd8a959edc1b7e4b67d"


def test_F2_partition_and_preemption(engines_gold):
    """in-engine PARTITION decisions + 212 preemptions."""
    g = engines_gold["F2"]
    out = run_case("rapid", LLAMA70B_LIKE, MI300X_LIKE, 2, SloSpec(itl_slo_us=50_000),
                   WorkloadSpec(qps=8.0, duration_s=120.0, seed=42, mean_prompt_tokens=2048, mean_output_tokens=1024,
                                sigma=0.0))
    _check(*out, g)
    assert g["preemptions"] == 212 and g["partition_decisions"] == 2842
    assert g["digest"] == "9c69c5bc10c6d2b03b0840c0138e10530d9ef90edbc6f73d6ae7d6ed67e1c0ec"


def test_F2_hybrid(engines_gold):
    out = run_case("hybrid-512", LLAMA70B_LIKE, MI300X_LIKE, 2, SloSpec(itl_slo_us=50_000),
                   WorkloadSpec(qps=8.0, duration_s=60.0, seed=42, mean_prompt_tokens=2048, mean_output_tokens=1024,
                                sigma=0.0))
    _check(*out, engines_gold["F2_hybrid512"])


def _tiny_items():
    return synthesize(WorkloadSpec(qps=4.0, duration_s=30.0, seed=0, mean_prompt_tokens=64,
                                   mean_output_tokens=16))[:64]


@pytest.mark.parametrize("case,label,params,pool,horizon", [
    ("tiny_rapid_2048", "rapid", None, None, None),
    ("tiny_rapid_32", "rapid", {"chunk_tokens": 32}, None, None),
    ("tiny_rapid_pool64", "rapid", {"chunk_tokens": 32}, 64, None),
    ("tiny_hybrid_64_pool64", "hybrid-64", None, 64, None),
    ("tiny_rapid_horizon", "rapid", None, 40, 8_000_000),
])
def test_tiny_full_records(engines_gold, case, label, params, pool, horizon):
    out = run_case(label, TINY, B200, 1, SloSpec(itl_slo_us=50_000), items=_tiny_items(), horizon=horizon,
                   engine_params=params, pool_blocks=pool)
    _check(*out, engines_gold[case], full=True)


@pytest.mark.parametrize("case,label", [("b200_8b_rapid", "rapid"), ("b200_8b_hybrid512", "hybrid-512")])
def test_b200_llama8b_trace(engines_gold, case, label):
    spec = WorkloadSpec(qps=48.0, duration_s=30.0, seed=42, mean_prompt_tokens=1024, mean_output_tokens=256, sigma=0.0)
    out = run_case(label, LLAMA8B, B200, 1, SloSpec(itl_slo_us=50_000), spec)
    _check(*out, engines_gold[case])


def test_costmodel_known_answers(cost_gold):
    p = CostParams()
    for name, tok, cu, conc, want in cost_gold["prefill"]:
        m, g = MODELS[name]
        assert prefill_time(tok, cu, m, g, p, conc) == want
    for name, b, kv, cu, conc, want in cost_gold["decode"]:
        m, g = MODELS[name]
        assert decode_time(b, kv, cu, m, g, p, conc) == want
    for name, pt, b, kv, mode, want in cost_gold["overlapped"]:
        m, g = MODELS[name]
        alloc = OVERALLOCATE if mode == "over" else AllocationDecision(AllocationMode.PARTITION, 0.6, 0.4)
        assert list(overlapped_times(pt, b, kv, alloc, m, g, p)) == want
    for name, pt, b, kv, want in cost_gold["hybrid"]:
        m, g = MODELS[name]
        assert hybrid_time(pt, b, kv, m, g, p) == want


def test_profiles_and_allocate(cost_gold):
    p = CostParams()
    profs = {}
    for key, lines in cost_gold["profiles"].items():
        name, slo_us = key.split("@")
        m, g = MODELS[name]
        prof = build_profile(m, g, p, int(slo_us))
        profs[key] = prof
        assert profile_lines(prof) == lines
    for name, slo_us, b, pt, want in cost_gold["allocate"]:
        m, g = MODELS[name]
        assert _dec(allocate(profs[f"{name}@{slo_us}"], b, pt, slo_us, m, g, p)) == want


def test_reference_frozen_timings():
    """Known answers quoted by the reference's own tests (test_costmodel.py:35-63)."""
    p = CostParams()
    g = MI300X_LIKE.aggregate(2) if False else MI300X_LIKE
    assert prefill_time(2048, 1.0, LLAMA70B_LIKE, g, p) == 219_366
    assert decode_time(1, 2048, 1.0, LLAMA70B_LIKE, g, p) == 26_602
