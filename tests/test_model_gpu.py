"""Decoder parity on the B200 against the fp32 CPU oracle (frozen cfg-1 tiny decoder,
same bf16-valued weights; oracle/llama_fp32.init_state "confident" init).

North-star bars, asserted on every generated token of every request:
  * greedy token ids EXACTLY equal to the oracle's greedy continuation (no near-tie band);
  * teacher-forced logits rel-L2 <= 2e-2 per step (bf16 GPU vs fp32 oracle).

The end-to-end runs serve SURVEY.md §8(d) cfg 1 exactly: the first 64 items of
synthesize(WorkloadSpec(qps=4, duration_s=30, seed=0, mean_prompt 64, mean_output 16)),
prompt ids torch.Generator().manual_seed(1000 + id), greedy, with chunk_tokens 2048 and 32,
plus a 64-block pool that forces preemption + recompute (time-compressed arrivals: at real
time the tiny model drains every request long before the next arrives, so the pool would
never fill), the same-engine hybrid comparator, and ARM re-splits captured lazily mid-run.
"""

import pytest
import torch

from oracle.llama_fp32 import Oracle, init_state
from paper_2601_11822_b200.model import DecoderWeights, Runner
from paper_2601_11822_b200.specs import ARCHS

pytestmark = pytest.mark.gpu
TOL = 2e-2  # north-star logits tolerance (relative L2 per row)


def rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return float((a - b).norm() / b.norm())


@pytest.fixture(scope="module")
def tiny():
    arch = ARCHS["tiny"]
    st = init_state(arch, seed=0)
    return arch, st, Oracle(arch, st), DecoderWeights.from_state(arch, st)


def cfg1_items():
    from paper_2601_11822_b200.traffic import WorkloadSpec, synthesize

    return synthesize(WorkloadSpec(qps=4.0, duration_s=30.0, seed=0, mean_prompt_tokens=64,
                                   mean_output_tokens=16))[:64]


def check_exact(orc, arch, engine, ex, *, label: str) -> dict:
    """Every finished request: GPU ids == oracle greedy ids, per-step logits rel-L2 <= TOL.

    The oracle runs teacher-forced on the GPU's tokens (one forward over prompt + gen[:-1]);
    argmax equality at every step makes the GPU sequence, by induction, the oracle's own
    free-running greedy continuation. Returns the margin / error statistics."""
    from paper_2601_11822_b200.traffic import prompt_token_ids

    done = [r for r in engine.requests if r.state.value == "finished"]
    worst_rel = worst_abs = 0.0
    min_margin = float("inf")
    ntok = 0
    for r in done:
        prompt = prompt_token_ids(r.id, r.prompt_tokens, arch.vocab).long()
        gen = ex.generated[r.id]
        assert len(gen) == r.output_tokens, (label, r.id)
        logits, _ = orc.forward(torch.cat([prompt, torch.tensor(gen[:-1], dtype=torch.long)]), 0, None)
        steps = logits[prompt.shape[0] - 1:]
        rows = ex.logits.get(r.id) if ex.record_logits else None
        assert rows is None or len(rows) == len(gen)
        for k, tok in enumerate(gen):
            ref = steps[k]
            want = int(ref.argmax())
            assert tok == want, (f"{label}: request {r.id} step {k}: GPU token {tok} != oracle greedy {want} "
                                 f"(first divergence)")
            if rows is None:  # ids only (the serving configuration: no logits copied back)
                ntok += 1
                continue
            e = rel(rows[k], ref)
            assert e <= TOL, (label, r.id, k, e)
            worst_rel = max(worst_rel, e)
            worst_abs = max(worst_abs, float((rows[k] - ref).abs().max()))
            top2 = torch.topk(ref, 2).values
            min_margin = min(min_margin, float(top2[0] - top2[1]))
            ntok += 1
    stats = {"requests": len(done), "tokens": ntok, "max_rel_l2": worst_rel, "max_abs_logit_err": worst_abs,
             "min_oracle_top1_margin": min_margin}
    print(label, stats)
    # the id check is decidable: the smallest oracle margin dwarfs the largest bf16 logit error
    if ex.record_logits:
        assert min_margin > 4 * worst_abs, stats
    return stats


def _runner(arch, w, nslots=4, nblocks=256):
    return Runner(w, num_blocks=nblocks, num_slots=nslots, max_blocks_per_seq=64, max_prefill_tokens=512,
                  max_decode_batch=16)


def test_prefill_chunks_then_decode_match_oracle(tiny):
    arch, st, orc, w = tiny
    r = _runner(arch, w)
    g = torch.Generator().manual_seed(5)
    P = 150
    prompt = torch.randint(0, arch.vocab, (P,), generator=g, dtype=torch.int32)
    pages = torch.randperm(256, generator=g)[:20].int()
    r.block_table[2, :20] = pages.cuda()
    # chunked prefill of positions 0..P-2 (Appendix C: last prompt token goes to decode)
    dev_ids = prompt.cuda()
    start = 0
    for ch in (64, 64, P - 1 - 128):
        lg = r.prefill(2, dev_ids[start:start + ch], start, num_sms=148, logits=True)
        start += ch
    torch.cuda.synchronize()
    ref_logits, _ = orc.forward(prompt.long(), 0, None)
    assert rel(lg[0], ref_logits[P - 2]) < TOL
    ref_ids, ref_steps = orc.greedy(prompt.long(), 6)
    r.last_tok[2] = int(prompt[P - 1])
    d = r.dec
    pos = P - 1
    for k in range(6):
        d.slot[:1] = 2
        d.pos[:1] = pos
        d.seq[:1] = pos + 1
        r.decode_body(1, num_sms=148)
        torch.cuda.synchronize()
        assert rel(d.logits[0], ref_steps[k]) < TOL, k
        assert int(d.out_ids[0]) == ref_ids[k], k
        assert int(r.last_tok[2]) == ref_ids[k]
        pos += 1


def test_batched_decode_rows_and_padding(tiny):
    arch, st, orc, w = tiny
    r = _runner(arch, w, nslots=8, nblocks=512)
    g = torch.Generator().manual_seed(9)
    lens = [5, 33, 70, 16]
    refs = []
    for s, L in enumerate(lens):
        prompt = torch.randint(0, arch.vocab, (L,), generator=g, dtype=torch.int32)
        r.block_table[s, :8] = torch.arange(s * 8, s * 8 + 8, dtype=torch.int32).cuda()
        r.prefill(s, prompt[: L - 1].cuda(), 0, num_sms=148)
        r.last_tok[s] = int(prompt[L - 1])
        lg, _ = orc.forward(prompt.long(), 0, None)
        refs.append(lg[-1])
    B, bucket = 4, 8
    d = r.dec
    d.slot[:bucket] = torch.tensor([0, 1, 2, 3] + [r.dummy_slot] * 4, dtype=torch.int32).cuda()
    d.pos[:bucket] = torch.tensor([L - 1 for L in lens] + [-1] * 4, dtype=torch.int32).cuda()
    d.seq[:bucket] = torch.tensor(lens + [0] * 4, dtype=torch.int32).cuda()
    r.decode_body(bucket, num_sms=148)
    torch.cuda.synchronize()
    for i in range(B):
        assert rel(d.logits[i], refs[i]) < TOL
        assert int(d.out_ids[i]) == int(torch.argmax(refs[i]))


def _serve(tiny, items, *, chunk, num_blocks=1024, engine="rapid", static_decode_sms=None, policy=None,
           prewarm=True, max_batch=32, record_logits=True):
    from paper_2601_11822_b200.arm import CostParams
    from paper_2601_11822_b200.engines.hybrid import HybridEngine
    from paper_2601_11822_b200.engines.rapid import RapidEngine
    from paper_2601_11822_b200.executor_b200 import B200Executor, HybridB200Executor
    from paper_2601_11822_b200.harness import run_items
    from paper_2601_11822_b200.slo import SloSpec
    from paper_2601_11822_b200.specs import b200_spec

    arch, st, orc, w = tiny
    model = arch.model_spec()
    slo = SloSpec(itl_slo_us=50_000)
    if engine == "hybrid":
        ex = HybridB200Executor(arch, weights=w, max_batch=max_batch, chunk_tokens=chunk, num_blocks=num_blocks,
                                max_context=1024, num_slots=128, record_logits=True)

        def factory():
            return HybridEngine(model, b200_spec(), CostParams(), slo, chunk_tokens=chunk, max_batch=max_batch,
                                executor=ex)
    else:
        ex = B200Executor(arch, weights=w, max_batch=max_batch, chunk_tokens=chunk, num_blocks=num_blocks,
                          max_context=1024, num_slots=128, static_decode_sms=static_decode_sms,
                          record_logits=record_logits)
        if prewarm:
            ex.warmup(sorted(policy.splits_used(), key=lambda d: -1 if d is None else d) if policy else None)

        def factory():
            return RapidEngine(model, b200_spec(), CostParams(), slo, chunk_tokens=chunk, max_batch=max_batch,
                               executor=ex, arm_policy=policy, record_decisions=True)
    res = run_items(engine, items, model, b200_spec(), CostParams(), slo, engine_factory=factory)
    return res, ex


@pytest.mark.parametrize("chunk,split", [(2048, 72), (32, 72), (32, None)])
def test_cfg1_trace_rapid_exact(tiny, chunk, split):
    """The full cfg-1 trace through RAPID on the real-time loop: static 72/76 green-context
    split or the reference ARM (OVERALLOCATE on both full-device streams)."""
    arch, st, orc, w = tiny
    items = cfg1_items()
    res, ex = _serve(tiny, items, chunk=chunk, static_decode_sms=split)
    assert sum(r.state.value == "finished" for r in res.engine.requests) == 64
    check_exact(orc, arch, res.engine, ex, label=f"rapid chunk={chunk} split={split}")
    ex.close()


def test_cfg1_trace_serving_config_ids_exact(tiny):
    """The serving configuration (no logits copied back): sampled ids are filed into
    `generated` off the critical path (at the loop's idle time, or when read); every token must
    still be the oracle's greedy id, with the green-context split."""
    arch, st, orc, w = tiny
    res, ex = _serve(tiny, cfg1_items(), chunk=32, static_decode_sms=72, record_logits=False)
    assert sum(r.state.value == "finished" for r in res.engine.requests) == 64
    check_exact(orc, arch, res.engine, ex, label="rapid serving config (ids only)")
    ex.close()


@pytest.mark.parametrize("record_logits", [True, False])
def test_cfg1_trace_preemption_pool_exact(tiny, record_logits):
    """cfg-1 prompts/outputs in a 64-block pool (SURVEY §8(d) cfg 1): RAPID preempts the most
    recent decoder on exhaustion (rapid.py:221-246) and re-prefills prompt + y1..y_{d-1};
    every token must still be the oracle's greedy id (also in the serving configuration, where
    the re-prefill reads ids filed off the critical path)."""
    from paper_2601_11822_b200.traffic import WorkloadItem

    arch, st, orc, w = tiny
    items = [WorkloadItem(it.arrival_us // 200, it.prompt_tokens, it.output_tokens) for it in cfg1_items()]
    res, ex = _serve(tiny, items, chunk=32, num_blocks=64, static_decode_sms=72, record_logits=record_logits)
    reqs = res.engine.requests
    assert sum(r.preemptions for r in reqs) >= 1, "the 64-block pool did not force a preemption"
    assert sum(r.state.value == "finished" for r in reqs) == 64
    check_exact(orc, arch, res.engine, ex, label=f"preemption pool ({sum(r.preemptions for r in reqs)} preemptions)")
    ex.close()


@pytest.mark.parametrize("chunk", [2048, 32])
def test_cfg1_trace_hybrid_exact(tiny, chunk):
    """Same-engine hybrid batching (fused decode rows + prefill chunk per iteration): first
    tokens come from the chunk that finishes each prompt (hybrid.py:144-155)."""
    arch, st, orc, w = tiny
    res, ex = _serve(tiny, cfg1_items(), chunk=chunk, engine="hybrid")
    assert sum(r.state.value == "finished" for r in res.engine.requests) == 64
    check_exact(orc, arch, res.engine, ex, label=f"hybrid chunk={chunk}")
    ex.close()


def _resplit_policy(max_batch):
    from paper_2601_11822_b200.arm import DEFAULT_BATCH_GRID, MeasuredArm, MeasuredProfile

    ladder = (16, 32, 48, 64)
    # decode step grows with the batch and shrinks with SMs: batch 1 fits the target on 16 SMs,
    # <= 2 on 32, <= 4 on 48, larger batches need 64
    dec = {str(d): {str(b): (48_000.0 if b > {16: 1, 32: 2, 48: 4, 64: 256}[d] else 1_000.0)
                    for b in DEFAULT_BATCH_GRID} for d in ladder}
    prof = MeasuredProfile({"model": "tiny", "ctx": 128, "chunk": 32, "total_sms": 148, "granularity": 8,
                            "batches": list(DEFAULT_BATCH_GRID), "decode_us": dec,
                            "prefill_us_per_token": {str(d): 10.0 + d / 10 for d in ladder},
                            "overalloc_decode_us": {str(b): 60_000.0 for b in DEFAULT_BATCH_GRID},
                            "overalloc_prefill_us_per_token": 9.0})
    return MeasuredArm(prof, 50_000, max_batch=max_batch, policy="slo-min")


@pytest.mark.parametrize("prewarm", [True, False])
def test_measured_arm_resplits_exact(tiny, prewarm):
    """RAPID driven by the measured-table ARM on a profile that moves the decode partition with
    the batch: launches hop between green-context splits mid-request. Without pre-warming,
    every (partition, bucket) graph is captured lazily while serving — the capture must not
    disturb the live step (executor_b200._capture parks the inputs)."""
    from paper_2601_11822_b200.traffic import WorkloadItem

    arch, st, orc, w = tiny
    policy = _resplit_policy(32)
    # a burst: prefills stay queued while the decode batch grows through the thresholds
    items = [WorkloadItem(1000 + 700 * i, 40 + (7 * i) % 50, 30 + (5 * i) % 20) for i in range(24)]
    res, ex = _serve(tiny, items, chunk=32, policy=policy, prewarm=prewarm)
    splits = {round(d.cu_fraction_decode * 148) for _, d in res.engine.decision_log if d.mode.value == "partition"}
    assert len(splits) >= 2, f"the profile should move the decode partition, saw {splits}"
    if not prewarm:
        assert ex.lazy_captures >= 2, ex.lazy_captures
    assert sum(r.state.value == "finished" for r in res.engine.requests) == len(items)
    check_exact(orc, arch, res.engine, ex, label=f"measured ARM re-splits prewarm={prewarm}")
    ex.close()
