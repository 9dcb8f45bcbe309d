"""Green-context quantisation of ARM decisions ("keep the decision
bit-exact and test the quantization separately"). specs.decode_sms_for maps
AllocationDecision (core.py:215-245) onto a decode partition of whole 8-SM granules."""

import pytest

from paper_2601_11822_b200.specs import (OVERALLOCATE, AllocationDecision, AllocationMode, SM_GRANULARITY,
                                         decode_sms_for)


def part(d_units, total=148):
    d = d_units / total
    return AllocationDecision(AllocationMode.PARTITION, (total - d_units) / total, d)


def test_overallocate_is_full_device():
    assert decode_sms_for(OVERALLOCATE, 148) is None


@pytest.mark.parametrize("units,want", [(1, 8), (8, 8), (9, 16), (38, 40), (72, 72), (73, 80), (95, 96),
                                        (136, 136), (137, 140), (140, 140), (147, 140)])
def test_partition_rounds_up_to_granule_and_leaves_prefill_one(units, want):
    got = decode_sms_for(part(units), 148)
    assert got == want
    assert got >= units or got == 148 - SM_GRANULARITY  # decode never gets fewer SMs than asked, unless capped
    assert 148 - got >= SM_GRANULARITY


def test_exact_multiples_survive_float_error():
    # cu fractions are k/148 floats: k*8/148*148 must not round up to the next granule
    for k in range(1, 18):
        assert decode_sms_for(part(8 * k), 148) == 8 * k


def test_every_fraction_on_the_reference_grid():
    # all 147 PARTITION decisions the reference ARM can emit (units of 1/num_cus)
    seen = set()
    for u in range(1, 148):
        s = decode_sms_for(part(u), 148)
        assert s % SM_GRANULARITY == 0 or s == 140
        assert 8 <= s <= 140
        assert s >= min(u, 140)
        seen.add(s)
    assert seen == set(range(8, 141, 8)) | {140}


def test_other_device_sizes():
    assert decode_sms_for(part(30, 132), 132) == 32
    assert decode_sms_for(part(131, 132), 132) == 124
