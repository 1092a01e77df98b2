"""Selector calibration from measured kernel latency (north-star item 4)."""

import json
import os

import pytest

import paper_2503_17924_b200 as wl
from paper_2503_17924_b200.calibrate import fit_profile

DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_2503_17924_b200", "data", "b200_llama7b_h32_d128.profile.json")


def test_fit_profile_recovers_piecewise_curve():
    # synthetic latency table from a known profile: throughput steps at q = 256
    truth = {0: 1e9, 256: 4e9}
    table = {}
    for q in (16, 64, 256, 1024):
        for kv in (2048, 8192):
            v = truth[256] if q >= 256 else truth[0]
            table[(q, kv)] = (-(-q // 128) * 128) * kv / v
    prof = fit_profile(table)
    assert prof.tile_size == 128 and prof.op_scale == 1.0
    assert prof.throughput(16) == pytest.approx(1e9)
    assert prof.throughput(300) == pytest.approx(4e9)
    assert prof.to_dict()["schema"] == "balsim.profile.v1"
    # the model reproduces every measured latency exactly
    for (q, kv), sec in table.items():
        assert wl.attention_kernel_latency(q, kv, prof) == pytest.approx(sec)


def test_shipped_b200_profile_is_valid():
    prof = wl.CostProfile.from_file(DATA)
    assert prof.tile_size == 128
    qs = [q for q, _ in prof.tflops_curve]
    assert qs[0] == 0 and qs == sorted(qs)
    assert json.load(open(DATA))["schema"] == "balsim.profile.v1"


@pytest.mark.gpu
def test_measure_and_select_with_calibrated_profile():
    from paper_2503_17924_b200.calibrate import measure
    table = measure(hq=4, hkv=4, d=64, q_grid=(16, 256), kv_grid=(1024,), iters=2, warmup=1)
    prof = fit_profile(table)
    assert all(s > 0 for s in table.values())
    mb = wl.MicroBatch([wl.Document(0, 96 * 1024)] + [wl.Document(i + 1, 1024) for i in range(32)])
    a = wl.adaptive_select(mb, 4, prof)       # runs the GPU selector under the measured profile
    assert a.strategy in (wl.ShardStrategy.PER_SEQUENCE, wl.ShardStrategy.PER_DOCUMENT)
