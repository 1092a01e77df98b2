"""BASELINE.json config 1 — the reference's own CPU-runnable case — end to end:
synthetic long-tail 8K sequences, 8 heads, D = 64, CP = 2, per-document
sharding, document-masked attention forward + backward.

For each of the 8 seed-0 sequences (`generate_synthetic_stream(SyntheticSpec(
8192, 8192), 0, 8)`, then `pad_for_cp`):

* the GPU shard builder's per-document assignment equals the oracle's
  restatement of `per_document_shard` (`/root/reference/pkg/src/balsim/
  sharding.py:113-141`) range for range;
* every CP rank's O, dQ and dK / dV partials from the tcgen05 kernels
  (pre-gathered K / V, the rank's local queries) agree with the fp32 CPU
  oracle (`oracle/attention_oracle.py::segment_attention_fwd_bwd`) within
  |got - ref| <= 2e-2 + 1e-2 |ref|; the strict max-abs is recorded;
* the CPU reference path of BASELINE.md §4 is timed beside it: the oracle's
  per-document shard and the per-rank fp32 fwd + bwd on all host threads
  (best of 3), next to the GPU per-rank kernel time (CUDA events, best of 3);
  per-rank seconds, TFLOP/s and max/mean are written as JSON lines to
  $WLB_CONFIG1_LOG when set (profiles/r02_config1.jsonl).
"""

import json
import os
import time

import pytest
import torch

import paper_2503_17924_b200 as wl
from paper_2503_17924_b200.attention import attn_backward, attn_forward, build_tiles
from oracle import attention_oracle as ao
from oracle import shard_oracle as so

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-2, 1e-2
T, HQ, HKV, D, CP = 8192, 8, 8, 64, 2


def _log(rec):
    path = os.environ.get("WLB_CONFIG1_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(rec) + "\n")


def _best(fn, reps=3, cuda=False):
    best = float("inf")
    for _ in range(reps):
        if cuda:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b) / 1e3)
        else:
            t0 = time.perf_counter()
            fn()
            best = min(best, time.perf_counter() - t0)
    return best


@pytest.mark.parametrize("seq", range(8))
def test_config1_sequence(seq):
    torch.set_num_threads(os.cpu_count())
    spec = wl.SyntheticSpec(context_window=T, tokens_per_global_batch=T)
    lengths = so.pad_lengths_for_cp([d.length for d in wl.generate_synthetic_stream(spec, 0, 8)[seq]],
                                    CP)
    total = sum(lengths)
    shard_s = _best(lambda: so.per_document(lengths, CP))
    ranges = so.per_document(lengths, CP)
    plan = wl.build_shard_plan([lengths], CP, "per_document")
    a = plan.assignment(0)
    assert [[(p, r.start, r.end) for p, r in w] for w in a.workers] == \
        [[tuple(x) for x in w] for w in ranges]

    g = torch.Generator().manual_seed(1000 + seq)
    mk = lambda h: torch.randn((total, h, D), generator=g).to(torch.bfloat16)
    q, k, v, do = mk(HQ), mk(HKV), mk(HKV), mk(HQ)
    dev = torch.device("cuda")
    kd, vd = k.to(dev), v.to(dev)
    rec = {"config": "config1", "seq": seq, "docs": len(lengths), "T": total, "cp": CP,
           "strategy": "per_document", "heads": [HQ, HKV], "head_dim": D,
           "cpu_threads": torch.get_num_threads(), "cpu_shard_ms": round(shard_s * 1e3, 4),
           "ranks": []}
    for w in range(CP):
        gidx, pos, ro = plan.rank_local(0, w)
        idx = gidx.long().cpu()
        ql, dol = q[idx].contiguous(), do[idx].contiguous()
        ref = ao.segment_attention_fwd_bwd(ql, k, v, dol, lengths, ranges[w])
        cpu_s = _best(lambda: ao.segment_attention_fwd_bwd(ql, k, v, dol, lengths, ranges[w]))
        tiles = build_tiles(ro, pos, lengths)
        qd, dod = ql.to(dev), dol.to(dev)

        def gpu():
            o_, lse_ = attn_forward(qd, kd, vd, tiles)
            return (o_, lse_) + attn_backward(qd, kd, vd, o_, lse_, dod, tiles)

        o, lse, dq, dk, dv = gpu()
        gpu_s = _best(gpu, cuda=True)
        errs = {}
        for name, got, want in (("o", o, ref[0]), ("dq", dq, ref[2]), ("dk", dk, ref[3]),
                                ("dv", dv, ref[4])):
            got, want = got.float().cpu(), want.float()
            excess = ((got - want).abs() - (ATOL + RTOL * want.abs())).max().item()
            errs[name] = round((got - want).abs().max().item(), 6)
            assert excess <= 0, f"seq {seq} rank {w} {name}: max abs {errs[name]:.3e}"
        assert (lse.cpu() - ref[1]).abs().max().item() < 1e-2
        pairs = so.worker_pairs(ranges[w])
        flops = 14.0 * D * HQ * pairs
        rec["ranks"].append({"rank": w, "pairs": pairs, "cpu_s": round(cpu_s, 4),
                             "cpu_tflops": round(flops / cpu_s / 1e12, 4),
                             "gpu_ms": round(gpu_s * 1e3, 4),
                             "gpu_tflops": round(flops / gpu_s / 1e12, 2), "max_abs": errs})
    for kind in ("cpu_s", "gpu_ms"):
        ts = [r[kind] for r in rec["ranks"]]
        rec[f"{kind.split('_')[0]}_imbalance"] = round(max(ts) / (sum(ts) / len(ts)), 4)
    _log(rec)
