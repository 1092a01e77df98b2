"""Pin the CPU oracle against the reference's own outputs (CPU only).

Golden vectors come from importing the reference package
(tests/golden/make_golden.py); `oracle/_ref` is the reference's Cython kernels
compiled from /root/reference by oracle/build.sh (skipped where absent).
"""

import ctypes
import glob
import importlib.util
import os

import numpy as np
import pytest
import torch

from conftest import ROOT, load_golden
from oracle import attention_oracle as ao
from oracle import shard_oracle as so

LIBORACLE = os.path.join(ROOT, "oracle", "liboracle.so")


def _oracle_lib():
    if not os.path.exists(LIBORACLE):
        pytest.skip("oracle/liboracle.so not built (run oracle/build.sh)")
    lib = ctypes.CDLL(LIBORACLE)
    P = ctypes.c_void_p
    lib.orc_kernel_latency_sum.restype = ctypes.c_double
    lib.orc_kernel_latency_sum.argtypes = [P, P, ctypes.c_longlong, ctypes.c_longlong, P, P,
                                           ctypes.c_longlong, ctypes.c_double]
    lib.orc_heuristic_fill.argtypes = [P, ctypes.c_longlong, ctypes.c_int, ctypes.c_longlong,
                                       ctypes.c_double, ctypes.c_double, P, P, P]
    lib.orc_sum_pair_counts.restype = ctypes.c_longlong
    lib.orc_sum_pair_counts.argtypes = [P, ctypes.c_longlong]
    lib.orc_range_pair_sum.restype = ctypes.c_longlong
    lib.orc_range_pair_sum.argtypes = [P, P, ctypes.c_longlong]
    return lib


def _i64(x):
    return np.ascontiguousarray(x, dtype=np.int64)


@pytest.mark.parametrize("name", ["sharding_random.json.gz", "sharding_synthetic.json.gz"])
def test_shard_oracle_matches_reference(name):
    for case in load_golden(name)["cases"]:
        lengths, cp = case["lengths"], case["cp"]
        assert [[list(r) for r in w] for w in so.per_sequence(lengths, cp)] == case["per_sequence"]
        assert [[list(r) for r in w] for w in so.per_document(lengths, cp)] == case["per_document"]
        cq, cv = [0, 256], [3.5e11, 7.0e11]
        for strat, key in ((so.SEQ, "lat_seq"), (so.DOC, "lat_doc")):
            a = so.shard(lengths, cp, strat)
            got = [so.worker_latency(a[w], 128, cq, cv, 70.0).hex() for w in range(cp)]
            assert got == case[key]
        choice = so.adaptive(lengths, cp, 128, cq, cv, 70.0)
        assert ("per_sequence" if choice == so.SEQ else "per_document") == case["adaptive"]


def test_shard_oracle_errors():
    with pytest.raises(ValueError):
        so.per_sequence([10], 2)
    with pytest.raises(ValueError):
        so.per_document([8], 0)


def test_c_oracle_kernels_match_reference_vectors():
    lib = _oracle_lib()
    g = load_golden("kernels.json.gz")
    for c in g["kernel_latency_sum"]:
        q, kv, cq = _i64(c["q"]), _i64(c["kv"]), _i64(c["cq"])
        cv = np.array([float.fromhex(x) for x in c["cv"]])
        got = lib.orc_kernel_latency_sum(q.ctypes.data, kv.ctypes.data, len(q), c["tile"],
                                         cq.ctypes.data, cv.ctypes.data, len(cq),
                                         float.fromhex(c["op"]))
        assert got.hex() == c["out"]
        assert so.kernel_latency_sum(c["q"], c["kv"], c["tile"], c["cq"], list(cv),
                                     float.fromhex(c["op"])).hex() == c["out"]
    for c in g["heuristic_fill"]:
        ls = _i64(c["lengths"])
        out = np.empty(len(ls), dtype=np.int32)
        scratch = np.empty(2 * c["n_mb"], dtype=np.int64)
        lib.orc_heuristic_fill(ls.ctypes.data, len(ls), c["n_mb"], c["l_max"], 2e-10, 2e-6,
                               scratch.ctypes.data, scratch[c["n_mb"]:].ctypes.data,
                               out.ctypes.data)
        assert out.tolist() == c["out"]
    for c in g["sum_pair_counts"]:
        ls = _i64(c["lengths"])
        assert lib.orc_sum_pair_counts(ls.ctypes.data, len(ls)) == c["out"]
    for c in g["range_pair_sum"]:
        s, e = _i64(c["s"]), _i64(c["e"])
        assert lib.orc_range_pair_sum(s.ctypes.data, e.ctypes.data, len(s)) == c["out"]
        assert sum(so.range_pairs(a, b) for a, b in zip(c["s"], c["e"])) == c["out"]


def test_reference_build_agrees_with_c_oracle():
    """oracle/_ref is the reference's own Cython source, compiled here."""
    found = glob.glob(os.path.join(ROOT, "oracle", "_ref", "_compiled*.so"))
    if not found:
        pytest.skip("oracle/_ref not built (reference absent)")
    spec = importlib.util.spec_from_file_location("_compiled", found[0])
    ref = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ref)
    lib = _oracle_lib()
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = int(rng.integers(0, 60))
        q = _i64(rng.integers(0, 9000, size=n))
        kv = _i64(q + rng.integers(1, 160000, size=n))
        cq = _i64([0, 256])
        cv = np.array([3.5e11, 7.0e11])
        a = ref.kernel_latency_sum(q, kv, 128, cq, cv, 70.0)
        b = lib.orc_kernel_latency_sum(q.ctypes.data, kv.ctypes.data, n, 128, cq.ctypes.data,
                                       cv.ctypes.data, 2, 70.0)
        assert a == b


def test_attention_oracle_shard_invariance():
    """CP-sharded doc-prefix attention == unsharded per-document causal attention
    (the known-answer property for attention)."""
    g = torch.Generator().manual_seed(0)
    lengths = [37, 5, 90, 1, 59]
    T = sum(lengths)
    cp = 2
    lengths = so.pad_lengths_for_cp(lengths, cp)
    T = sum(lengths)
    q = torch.randn(T, 4, 16, generator=g)
    k = torch.randn(T, 2, 16, generator=g)
    v = torch.randn(T, 2, 16, generator=g)
    full, _ = ao.doc_causal_attention(q, k, v, lengths)
    for strat in (so.SEQ, so.DOC):
        a = so.shard(lengths, cp, strat)
        for w in range(cp):
            gidx, _ = so.local_layout(lengths, a[w])
            out, _ = ao.segment_attention(q[gidx], k, v, lengths, a[w])
            assert torch.allclose(out, full[gidx], atol=1e-5)


def _sdpa_doc_causal(q, k, v, do, lengths):
    """Independent reference: torch's own is_causal SDPA per document (GQA by
    repeat_interleave), fwd + autograd bwd, fp32."""
    import torch.nn.functional as F
    q = q.clone().requires_grad_(True)
    k = k.clone().requires_grad_(True)
    v = v.clone().requires_grad_(True)
    hq, hkv = q.shape[1], k.shape[1]
    outs, s0 = [], 0
    for L in lengths:
        qs = q[s0:s0 + L].transpose(0, 1)
        ks = k[s0:s0 + L].repeat_interleave(hq // hkv, dim=1).transpose(0, 1)
        vs = v[s0:s0 + L].repeat_interleave(hq // hkv, dim=1).transpose(0, 1)
        outs.append(F.scaled_dot_product_attention(qs, ks, vs, is_causal=True).transpose(0, 1))
        s0 += L
    out = torch.cat(outs, 0)
    out.backward(do)
    return out.detach(), q.grad, k.grad, v.grad


def test_attention_oracle_matches_independent_sdpa():
    """Both oracle forms (autograd and the query-blocked explicit backward used
    at config scale) against torch's is_causal SDPA per document, every CP rank
    under both strategies: the concatenated per-rank outputs and the rank-summed
    dK/dV partials equal the unsharded per-document result."""
    g = torch.Generator().manual_seed(3)
    hq, hkv, d = 8, 2, 32
    for cp in (1, 2, 4):
        lengths = so.pad_lengths_for_cp([130, 1, 67, 300, 9, 2], cp)
        T = sum(lengths)
        q, do = torch.randn(T, hq, d, generator=g), torch.randn(T, hq, d, generator=g)
        k, v = torch.randn(T, hkv, d, generator=g), torch.randn(T, hkv, d, generator=g)
        ro, rdq, rdk, rdv = _sdpa_doc_causal(q, k, v, do, lengths)
        for strat in (so.SEQ, so.DOC):
            a = so.shard(lengths, cp, strat)
            dk_sum, dv_sum = torch.zeros_like(k), torch.zeros_like(v)
            for w in range(cp):
                idx = torch.tensor(so.local_layout(lengths, a[w])[0], dtype=torch.long)
                auto = ao.segment_attention_fwd_bwd(q[idx], k, v, do[idx], lengths, a[w])
                blk = ao.segment_attention_fwd_bwd_blocked(q[idx], k, v, do[idx], lengths, a[w],
                                                           block=48)
                for x, y in zip(auto, blk):
                    assert torch.allclose(x, y, atol=2e-5, rtol=1e-5)
                for x, y in zip((blk[0], blk[2]), (ro[idx], rdq[idx])):
                    assert torch.allclose(x, y, atol=2e-5, rtol=1e-5)
                dk_sum += blk[3]
                dv_sum += blk[4]
            assert torch.allclose(dk_sum, rdk, atol=2e-5, rtol=1e-5)
            assert torch.allclose(dv_sum, rdv, atol=2e-5, rtol=1e-5)
