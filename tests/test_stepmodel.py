"""Measured attention latency into the reference's pipeline step model
(paper_2503_17924_b200/stepmodel.py).

Golden values come from the reference's own `pipeline.py` / `packing.py`
(tests/golden/make_golden.py::pipeline_model)."""

import gzip
import json
import os

import pytest

import paper_2503_17924_b200 as wl
from paper_2503_17924_b200 import stepmodel as sm

GOLD = os.path.join(os.path.dirname(__file__), "golden", "pipeline_model.json.gz")


def _gold():
    with gzip.open(GOLD) as fh:
        return json.load(fh)


def test_pp_critical_path_matches_reference():
    for case in _gold()["paths"]:
        stages = [sm.StageLatency(float.fromhex(f), float.fromhex(b)) for f, b in case["stages"]]
        assert sm.pp_critical_path(stages, case["pp"]).hex() == case["out"]
    with pytest.raises(ValueError):
        sm.pp_critical_path([], 0)


def test_imbalance_latency_matches_reference():
    prof = wl.CostProfile()
    for case in _gold()["imbalance_latency"]:
        mbs = [wl.MicroBatch([wl.Document(i, x) for i, x in enumerate(ls)]) for ls in case["mbs"]]
        assert wl.imbalance_degree_latency(mbs, len(mbs), prof).hex() == case["out"]


def test_measured_stage_formula():
    prof = wl.CostProfile()
    par = wl.ParallelismConfig(context_window=32768, cp=4, pp=2)
    st = sm.measured_stage_latency(0.010, 0.025, 8192, par, prof)
    lin = wl.linear_workload_latency(8192, prof)
    assert st.forward == (0.010 + lin) / 2
    assert st.backward == (0.025 + prof.backward_ratio * lin) / 2
    assert st.round_trip == st.forward + st.backward


def test_measured_step_report():
    prof = wl.CostProfile()
    par = wl.ParallelismConfig(context_window=32768, cp=2, pp=4)
    mbs = [[4096, 4096], [8000, 192], [2048] * 4]
    rep = sm.measured_step_report(7, mbs, ["per_document", "per_sequence", "per_sequence"],
                                  [0.01, 0.02, 0.005], [0.03, 0.05, 0.012], par, prof)
    assert rep.iteration == 7 and rep.microbatch_tokens == [8192, 8192, 8192]
    assert rep.microbatch_attention_pairs == [wl.attention_workload(x) for x in mbs]
    stages = [sm.StageLatency(f, b) for f, b in zip(rep.forward, rep.backward)]
    assert rep.replica_paths == [sm.pp_critical_path(stages, 4)]
    assert rep.dp_step_latency == rep.replica_paths[0]
    assert rep.event_makespan is None and rep.strategy_choices[0] == "per_document"


@pytest.mark.gpu
def test_stage_latency_for_assignment_matches_reference():
    """Modelled stage cost through the GPU builder/selector: bit-exact."""
    prof = wl.CostProfile()
    for case in _gold()["stages"]:
        mb = wl.MicroBatch([wl.Document(i, x) for i, x in enumerate(case["lengths"])])
        par = wl.ParallelismConfig(context_window=65536, cp=case["cp"], pp=case["pp"])
        st = sm.microbatch_stage_latency(mb, par, prof, case["policy"])
        assert (st.forward.hex(), st.backward.hex()) == (case["forward"], case["backward"]), case


@pytest.mark.gpu
def test_measure_attention_latency_single_gpu():
    import torch
    from paper_2503_17924_b200.cp import build_cp_shards
    lengths = [[3000, 1000, 96], [4096]]
    shards = build_cp_shards(lengths, 1, 0, "adaptive")
    dev = torch.device("cuda")
    inputs = [tuple(torch.randn(sum(ls), 4, 128, device=dev, dtype=torch.bfloat16)
                    for _ in range(4)) for ls in lengths]
    fwd, bwd = sm.measure_attention_latency(shards, inputs, reps=3)
    assert len(fwd) == len(bwd) == 2 and all(x > 0 for x in fwd + bwd)
    par = wl.ParallelismConfig(context_window=8192, cp=1, pp=2)
    rep = sm.measured_step_report(0, lengths, [s.strategy for s in shards], fwd, bwd, par,
                                  wl.CostProfile())
    assert rep.dp_step_latency > 0
