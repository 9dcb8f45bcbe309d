"""Measured-table ARM (arm.MeasuredProfile / MeasuredArm) on a synthetic profile.

The tables mimic profiler.py output: decode step time falls with decode SMs and
grows with batch; the prefill side's per-token time grows as decode takes SMs.
"""

import pytest

from paper_2601_11822_b200.arm import (DEFAULT_BATCH_GRID, MeasuredArm, MeasuredProfile, decode_sms_of,
                                       profile_lines)
from paper_2601_11822_b200.specs import AllocationMode

LADDER = (16, 24, 32, 40, 48, 56, 64, 72, 88, 104, 120, 136)


def synth(total=148):
    dec, pre = {}, {}
    for d in LADDER:
        # weights 15 ms-equivalent at 16 SMs shrinking with SMs; KV term linear in batch
        dec[str(d)] = {str(b): round((3000 + 60 * b) * 72 / min(d, 96), 1) for b in DEFAULT_BATCH_GRID}
        pre[str(d)] = round(20.0 * 76 / (total - d), 3)
    return {"model": "synthetic", "ctx": 1152, "chunk": 2048, "total_sms": total, "granularity": 8,
            "batches": list(DEFAULT_BATCH_GRID), "decode_us": dec, "prefill_us_per_token": pre,
            "overalloc_decode_us": {str(b): round(1.6 * (3000 + 60 * b), 1) for b in DEFAULT_BATCH_GRID},
            "overalloc_prefill_us_per_token": 14.0}


def test_profile_lines_match_reference_format():
    mp = MeasuredProfile(synth())
    prof = mp.to_profile(50_000)
    lines = profile_lines(prof)
    assert len(lines) == len(DEFAULT_BATCH_GRID)
    for ln, b in zip(lines, DEFAULT_BATCH_GRID):
        parts = ln.split(",")
        assert int(parts[0]) == b
        frac = float(parts[1])
        # smallest ladder partition whose step fits 0.9 x SLO
        want = next((d for d in LADDER if mp.decode_us(d, b) <= 45_000), None)
        if want is None:
            assert parts[2] == "saturated"
        else:
            assert abs(frac - want / 148) < 1e-6


def test_idle_phase_overallocates():
    arm = MeasuredArm(MeasuredProfile(synth()), 50_000)
    assert arm.decide(0, 4096, 0.25).mode is AllocationMode.OVERALLOCATE
    assert arm.decide(128, 0, 0.25).mode is AllocationMode.OVERALLOCATE


def test_balanced_split_meets_slo_and_balances():
    mp = MeasuredProfile(synth())
    arm = MeasuredArm(mp, 50_000, max_batch=256, policy="balanced")
    for b in (16, 64, 128, 256):
        d = decode_sms_of(arm.decide(b, 2048, 0.25), 148)
        assert mp.decode_us(d, b) <= 45_000
    # more output per prompt token -> decode side needs more SMs (never fewer)
    lo = decode_sms_of(arm.decide(128, 2048, 0.05), 148)
    hi = decode_sms_of(arm.decide(128, 2048, 1.0), 148)
    lo_v = 148 if lo is None else lo
    hi_v = 148 if hi is None else hi
    assert lo_v <= hi_v


def test_slo_min_is_reference_rule():
    mp = MeasuredProfile(synth())
    arm = MeasuredArm(mp, 50_000, policy="slo-min")
    prof = mp.to_profile(50_000)
    for b in DEFAULT_BATCH_GRID:
        dec = arm.decide(b, 1024, 0.25)
        if mp.decode_us(None, b) <= 50_000:
            assert dec.mode is AllocationMode.OVERALLOCATE
        else:
            e = prof.lookup(b)
            assert dec.mode is AllocationMode.PARTITION
            assert decode_sms_of(dec, 148) == (LADDER[-1] if e.saturated else round(e.cu_fraction * 148))


def test_splits_used_covers_decisions():
    arm = MeasuredArm(MeasuredProfile(synth()), 50_000)
    used = arm.splits_used()
    for b in DEFAULT_BATCH_GRID:
        assert decode_sms_of(arm.decide(b, 1, 0.25), 148) in used


def test_bad_policy():
    with pytest.raises(ValueError):
        MeasuredArm(MeasuredProfile(synth()), 50_000, policy="nope")


def test_adaptive_policy_walks_with_queue_feedback():
    mp = MeasuredProfile(synth())
    arm = MeasuredArm(mp, 50_000, max_batch=256, policy="adaptive")
    d0 = decode_sms_of(arm.decide(128, 2048, 0.25), 148)
    assert d0 == arm._balanced(128, 0.25)
    # decode-bound windows (decoders waiting beyond max_batch) move decode up one granule
    for _ in range(arm.WINDOW):
        arm.observe(20_000, 256, 5, 3)
    d1 = decode_sms_of(arm.decide(256, 2048, 0.25), 148)
    assert d1 is not None and d1 > d0
    # a standing prefill queue with decode slack moves one granule back
    for _ in range(arm.WINDOW):
        arm.observe(15_000, 128, 0, 4)
    d2 = decode_sms_of(arm.decide(128, 2048, 0.25), 148)
    assert d2 < d1
    # every split the walk can reach is pre-captured
    i = mp.ladder.index(d0)
    assert set(mp.ladder[max(0, i - arm.SPAN):i + arm.SPAN + 1]) <= arm.splits_used()
    # idle phases still overallocate
    assert arm.decide(0, 100, 0.25).mode is AllocationMode.OVERALLOCATE


@pytest.mark.parametrize("name", ["llama3.1-8b_ctx1152_chunk1023.json", "qwen2.5-14b_ctx8256.json"])
def test_committed_b200_profiles(name):
    """The measured tables bench.py serves with by default: well-formed, monotone in the
    ways the policy relies on, and every decision they drive fits the SLO target."""
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(__file__)), "profiles", "arm", name)
    mp = MeasuredProfile.load(path)
    assert mp.total == 148 and len(mp.ladder) >= 8
    # more decode SMs never make the (measured) step much slower
    for b in mp.batches:
        steps = [mp.decode_us(d, b) for d in mp.ladder]
        assert all(steps[i + 1] <= steps[i] * 1.15 for i in range(len(steps) - 1)), (b, steps)
    for policy in ("balanced", "adaptive", "slo-min"):
        arm = MeasuredArm(mp, 50_000, max_batch=256, policy=policy)
        for b in mp.batches:
            d = decode_sms_of(arm.decide(b, 2048, 0.25), 148)
            if policy != "slo-min" and d is not None and arm.candidates(b):
                assert mp.decode_us(d, b) <= arm.target
    lines = profile_lines(mp.to_profile(50_000))
    assert len(lines) == len(mp.batches)


def test_calibrate_recovers_cost_model_parameters():
    """Tables generated by the reference decode_time itself (known bandwidth factor, plateau
    and overhead) are fitted back by arm.calibrate with ~zero error."""
    import dataclasses

    from paper_2601_11822_b200.arm import CostParams, calibrate, decode_time, prefill_time
    from paper_2601_11822_b200.specs import ARCHS, b200_spec

    model = ARCHS["llama3.1-8b"].model_spec()
    gpu0 = b200_spec()
    g = dataclasses.replace(gpu0, hbm_bandwidth=gpu0.hbm_bandwidth * 0.8, peak_flops=gpu0.peak_flops * 0.9)
    p = dataclasses.replace(CostParams(), decode_plateau_fraction=0.5, fixed_iteration_overhead_us=1000.0)
    ctx, chunk = 1152, 1024
    dec = {str(d): {str(b): float(decode_time(b, b * ctx, d / 148, model, g, p, concurrent=True))
                    for b in DEFAULT_BATCH_GRID} for d in LADDER}
    pre = {str(d): prefill_time(chunk, (148 - d) / 148, model, g, p, concurrent=True) / chunk for d in LADDER}
    mp = MeasuredProfile({"model": "x", "ctx": ctx, "chunk": chunk, "total_sms": 148, "granularity": 8,
                          "batches": list(DEFAULT_BATCH_GRID), "decode_us": dec, "prefill_us_per_token": pre,
                          "overalloc_decode_us": {str(b): 30_000.0 for b in DEFAULT_BATCH_GRID},
                          "overalloc_prefill_us_per_token": 15.0})
    res = calibrate(mp, model, gpu0, CostParams())
    assert abs(res["fit"]["hbm_bandwidth_factor"] - 0.8) < 1e-9
    assert abs(res["fit"]["decode_plateau_fraction"] - 0.5) < 1e-9
    assert res["fit"]["fixed_iteration_overhead_us"] == 1000.0
    assert abs(res["fit"]["peak_flops_factor"] - 0.9) < 0.03
    assert res["partition_decode_rel_err"]["max"] < 1e-3


def test_committed_cost_fits():
    """The refits written from the measured tables: partition decode steps within a few % (median),
    and the reference OVERALLOCATE model far below the measured contended steps."""
    import json
    import os

    for name in ("llama3.1-8b_costfit.json", "qwen2.5-14b_costfit.json"):
        with open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "profiles", "arm", name)) as fh:
            fit = json.load(fh)
        assert fit["partition_decode_rel_err"]["median"] < 0.1
        assert fit["overallocate_decode_rel_err"]["median"] < -0.3


def test_feedback_policy_alternates_on_backlog():
    """The backlog-buffered policy: prefill-heavy split while the ready-decoder backlog is
    small, decode-heavy once it passes FB_BACKLOG_HI, back below FB_BACKLOG_LO (hysteresis);
    both ends fit the SLO target at the batch cap and are pre-captured."""
    mp = MeasuredProfile(synth())
    arm = MeasuredArm(mp, 50_000, max_batch=256, policy="feedback")
    lo, hi = arm._hull_pair(0.25)
    assert lo <= hi
    for d in (lo, hi):
        assert mp.decode_us(d, 256) <= arm.target
        assert d in arm.splits_used()
    d0 = decode_sms_of(arm.decide(256, 2048, 0.25), 148)
    assert d0 == lo
    for _ in range(arm.FB_WINDOW):
        arm.observe(20_000, 256, arm.FB_BACKLOG_HI, 3)
    assert decode_sms_of(arm.decide(256, 2048, 0.25), 148) == hi
    for _ in range(arm.FB_WINDOW):  # inside the hysteresis band: stays decode-heavy
        arm.observe(20_000, 256, (arm.FB_BACKLOG_HI + arm.FB_BACKLOG_LO) // 2, 3)
    assert decode_sms_of(arm.decide(256, 2048, 0.25), 148) == hi
    for _ in range(arm.FB_WINDOW):
        arm.observe(20_000, 256, 0, 3)
    assert decode_sms_of(arm.decide(256, 2048, 0.25), 148) == lo
    assert arm.decide(0, 100, 0.25).mode is AllocationMode.OVERALLOCATE


def test_feedback_hull_beats_single_split_on_committed_profile():
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(__file__)), "profiles", "arm",
                        "llama3.1-8b_ctx1152_chunk1023.json")
    mp = MeasuredProfile.load(path)
    arm = MeasuredArm(mp, 50_000, max_batch=256, policy="feedback")
    lo, hi = arm._hull_pair(0.25)

    def pt(d):
        return 256 / mp.decode_us(d, 256), 0.25 / mp.prefill_us_per_token(d, 256)

    (xl, yl), (xh, yh) = pt(lo), pt(hi)
    a = (yl - xl) / ((yl - xl) + (xh - yh))
    hull = xl + a * (xh - xl)
    single = max(min(*pt(d)) for d in arm.candidates(256) if d is not None)
    assert lo < hi and hull > single
