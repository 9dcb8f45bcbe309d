"""bench.partition_bound: decode attention's in-situ rate against min(HBM, SMs x 64 B x clock)."""

import pytest

import bench


def test_partition_bound_per_partition_and_time_weighted():
    # 32 SMs at 1,410 MHz: 32 x 64 B x 1.41 GHz = 2,887.7 GB/s (below HBM); 64 SMs: 5,775.4
    by_sms = {"32": {"gbs": 2746.2, "bytes": 2746.2e6 * 2.0, "ms": 2.0},
              "64": {"gbs": 4809.8, "bytes": 4809.8e6 * 3.0, "ms": 3.0}}
    r = bench.partition_bound(by_sms, 1410.0, 6546.9)
    assert r["by_decode_sms"]["32"]["bound_gbs"] == pytest.approx(2887.7, abs=0.1)
    assert r["by_decode_sms"]["64"]["bound_gbs"] == pytest.approx(5775.4, abs=0.1)
    assert r["by_decode_sms"]["32"]["frac"] == pytest.approx(2746.2 / 2887.68, abs=1e-3)
    t_bound = 2746.2e6 * 2.0 / 2887.68e6 + 4809.8e6 * 3.0 / 5775.36e6
    assert r["frac"] == pytest.approx(t_bound / 5.0, abs=1e-3)


def test_partition_bound_caps_at_hbm_and_handles_missing_clock():
    r = bench.partition_bound({"148": {"gbs": 6900.0, "bytes": 6.9e9, "ms": 1.0}}, 1965.0, 6546.9)
    assert r["by_decode_sms"]["148"]["bound_gbs"] == pytest.approx(6546.9)
    assert bench.partition_bound({"32": {"gbs": 1.0, "bytes": 1.0, "ms": 1.0}}, None, 6546.9) is None
    assert bench.partition_bound({}, 1410.0, 6546.9) is None
