"""Host-side API and C-ABI checks (CPU only, no GPU compute)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden
import paper_2503_17924_b200 as wl
from paper_2503_17924_b200 import _native


def test_abi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "wlbcp.h")).read()
    declared = set(re.findall(r"\b(wlb_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.SIGNATURES), "binding table out of sync with wlbcp.h"
    assert _native.lib().wlb_abi_version() == 1


def test_library_has_sm100a_tensor_core_code():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out or "UTCQMMA" in out          # tcgen05.mma
    assert "UTMALDG" in out                               # TMA loads
    assert "LDTM" in out                                  # tcgen05.ld


def test_heuristic_fill_native_matches_reference():
    for c in load_golden("kernels.json.gz")["heuristic_fill"]:
        out = wl.heuristic_fill(c["lengths"], c["n_mb"], c["l_max"], 2e-10, 2e-6)
        assert out.tolist() == c["out"]


def test_packer_config5_trace_matches_reference():
    """HeuristicPacker + pad_for_cp reproduce the reference's config-5 stream."""
    g = load_golden("packer_config5.json.gz")["iterations"]
    spec = wl.SyntheticSpec(context_window=131072, tokens_per_global_batch=64 * 131072)
    stream = wl.generate_synthetic_stream(spec, seed=0, n_batches=len(g))
    packer = wl.HeuristicPacker(wl.OutlierQueueSet((32768, 98304)), 64, 163840, wl.CostProfile())
    filler = wl._FillerIds()
    for it, batch in enumerate(stream):
        plan = packer.feed(batch, it)
        exp = g[it]
        for mb, e in zip(plan.microbatches, exp["microbatches"]):
            padded = wl.pad_for_cp(mb, 8, filler, it)
            assert [d.id for d in padded.docs] == e["ids"]
            assert padded.lengths() == e["lengths"]
            assert [d.arrival_batch for d in padded.docs] == e["arrivals"]
        assert [d.id for d in plan.carried_over] == exp["carried"]
        assert sorted([k, v] for k, v in plan.delayed_tokens.items()) == exp["delayed"]
        assert packer.queues.depths() == exp["depths"]


def test_packer_streaming_trace_hand_example():
    """test_packing.py:243-271 of the reference."""
    mk = lambda ls, arrival=0, first=0: [wl.Document(first + i, x, arrival) for i, x in enumerate(ls)]
    packer = wl.HeuristicPacker(wl.OutlierQueueSet((10,)), 2, 16, wl.CostProfile())
    plan0 = packer.feed(mk([12, 3, 3, 2]), 0)
    assert [mb.lengths() for mb in plan0.microbatches] == [[3, 2], [3]]
    plan1 = packer.feed(mk([11, 4, 4, 3], 1, 4), 1)
    assert [mb.lengths() for mb in plan1.microbatches] == [[12, 4], [11, 4]]
    assert [d.id for d in plan1.carried_over] == [7]
    flushed = packer.flush(2)
    assert [mb.lengths() for mb in flushed[0].microbatches] == [[3], []]
    with pytest.raises(wl.ConfigError):
        wl.HeuristicPacker(wl.OutlierQueueSet([20]), 2, 16, wl.CostProfile())


def test_synthetic_generator_matches_reference():
    g = load_golden("synthetic_streams.json.gz")["streams"]
    for w in ("8192", "32768", "131072"):
        s = wl.generate_synthetic_stream(wl.SyntheticSpec(int(w), int(w)), 0, 8)
        assert [[[d.id, d.length, d.arrival_batch] for d in b] for b in s] == g[w]


def test_workload_and_profile_semantics(tmp_path):
    p = wl.CostProfile()
    assert wl.attention_workload([4]) == 10 and wl.attention_workload([]) == 0
    assert wl.range_attention_workload(8, wl.TokenRange(4, 8)) == 26
    with pytest.raises(ValueError):
        wl.range_attention_workload(8, wl.TokenRange(4, 9))
    with pytest.raises(ValueError):
        wl.TokenRange(3, 3)
    assert wl.attention_kernel_latency(0, 5, p) == 0.0
    with pytest.raises(ValueError):
        wl.attention_kernel_latency(64, 0, p)
    assert wl.attention_kernel_latency(1, 1024, p) == wl.attention_kernel_latency(128, 1024, p)
    assert wl.attention_kernel_latency(129, 1000, p) == p.op_scale * (256 * 1000) / p.throughput(129)
    with pytest.raises(wl.ConfigError):
        wl.CostProfile(tflops_curve=((1, 1e11),))
    with pytest.raises(wl.ConfigError):
        wl.CostProfile.from_dict({"bogus": 1})
    prof = wl.CostProfile(attn_coeff=3e-10, op_scale=55.0, tflops_curve=((0, 1e11), (512, 4e11)))
    prof.to_file(tmp_path / "p.json")
    assert wl.CostProfile.from_file(tmp_path / "p.json") == prof


def test_pad_for_cp():
    f = wl._FillerIds()
    mb = wl.MicroBatch([wl.Document(0, 13)])
    out = wl.pad_for_cp(mb, 4, f, 2)
    assert out.lengths() == [13, 3] and out.docs[-1].id == -1_000_000
    assert out.docs[-1].arrival_batch == 2
    assert wl.pad_for_cp(wl.MicroBatch([wl.Document(0, 16)]), 4, f, 0).lengths() == [16]
    assert wl.pad_for_cp(mb, 4, f, 0).docs[-1].id == -1_000_001


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    mb = wl.MicroBatch([wl.Document(0, 16)])
    with pytest.raises(wl.NativeError):
        wl.per_document_shard(mb, 2)
    # validation still happens first, exactly like the reference
    with pytest.raises(ValueError):
        wl.per_document_shard(wl.MicroBatch([wl.Document(0, 9)]), 2)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2503_17924_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|oracle/)", src), f


def test_abi_argument_validation_without_gpu():
    """Entry points validate sizes before touching the device and report
    WLB_EINVAL (-> ValueError in the wrappers), as the reference's callers
    raise ValueError for bad arguments (sharding.py:77-83)."""
    from paper_2503_17924_b200 import _native
    lib = _native.lib()
    # head dim not a multiple of 4, non-positive base
    assert lib.wlb_qkv_rope(None, None, None, None, None, 8, 4, 2, 6, 1e4, None) == _native.WLB_EINVAL
    assert lib.wlb_qkv_rope(None, None, None, None, None, 8, 4, 2, 128, 1.0, None) == _native.WLB_EINVAL
    assert b"rope" in lib.wlb_last_error()
    # Tl == 0 is a no-op
    assert lib.wlb_qkv_rope(None, None, None, None, None, 0, 4, 2, 128, 1e4, None) == _native.WLB_OK
    # attention: unsupported head dim / GQA ratio
    assert lib.wlb_attn_fwd(None, None, None, None, None, None, None, 1, None, 8, 8, 4, 4, 96,
                            0.1, None) == _native.WLB_EINVAL
    assert lib.wlb_attn_bwd(None, None, None, None, None, None, None, None, None, None, None, 1,
                            None, 8, 8, 6, 4, 128, 0.1, None, None) == _native.WLB_EINVAL
