"""bench.py contract pieces that run without a GPU: the workload table behind
`metric`/`config` (BASELINE.json configs 2-4) and the reference arm's rank
rule (rank 0 alone prints; the other ranks exit without work)."""

import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.path.insert(0, ROOT)
    spec.loader.exec_module(mod)
    return mod


def test_workloads_match_baseline_configs():
    b = _bench()
    w1 = b._workload(1)
    assert (w1["window"], w1["hq"], w1["hkv"], w1["d"], w1["cp"]) == (32768, 32, 32, 128, 1)
    for n in (2, 4, 8):
        w = b._workload(n)
        assert (w["window"], w["hq"], w["hkv"], w["d"], w["cp"]) == (131072, 32, 32, 128, n)
        assert w["window"] % (2 * n) == 0          # sharding needs T divisible by 2*cp
        g = b._workload(n, "llama70b-gqa")
        assert (g["hq"], g["hkv"], g["d"]) == (64, 8, 128) and g["name"].startswith("llama70b-gqa")


def test_synthetic_lengths_fill_each_sequence():
    b = _bench()
    for window in (32768, 131072):
        ls = b._lengths(window)
        assert len(ls) == b.N_SEQ
        assert all(sum(x) == window and min(x) >= 1 for x in ls)


def test_reference_arm_non_zero_ranks_do_nothing(capsys):
    b = _bench()

    class A:
        steps, warmup = 1, 0
    b.run_reference(A(), world=4, rank=2)
    assert capsys.readouterr().out == ""


def test_clock_summary_flags_throttle_reasons():
    """`clocks` keeps the busy-clock median and every throttle reason seen
    (the contract rejects hw_slowdown / thermal runs; sw_power_cap is noted)."""
    b = _bench()
    c = b.ClockSampler(0, 0)
    with c:
        pass
    assert c.summary()["samples"] == 0
    c.lines = ["1800, 1965, Not Active, Not Active, Not Active, Active",
               "1700, 1965, Not Active, Active, Not Active, Not Active",
               "300, 1965, Not Active, Not Active, Not Active, Not Active",
               "garbage"]
    s = c.summary()
    assert s["samples"] == 3 and s["sm_max_mhz"] == 1965.0
    assert s["sm_mhz"] == 1750.0                    # idle 300 MHz sample excluded
    assert s["reasons"] == ["hw_thermal_slowdown", "sw_power_cap"]


def test_fixed_128k_workload_for_strong_scaling():
    """--workload 128k keeps the same 8 x 128K sequences at every N (CP = N,
    N = 1 included), so N = 1/2/4/8 measure fixed total work."""
    b = _bench()
    for n in (1, 2, 4, 8):
        w = b._workload(n, workload="128k")
        assert (w["window"], w["cp"]) == (131072, n)


def test_gpus_must_match_world_size(monkeypatch):
    """Under torchrun, --gpus N must equal WORLD_SIZE (no silent N=1 run)."""
    b = _bench()
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    import pytest
    with pytest.raises(SystemExit, match="WORLD_SIZE=2"):
        b.main()


def test_host_steps_times_the_reference_selector():
    b = _bench()
    ms = b._host_steps(b._lengths(8192)[:2], 2)
    assert ms > 0
