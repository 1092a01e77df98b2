"""Calibrate the CP strategy selector from MEASURED B200 kernel latency.

North-star item 4: the adaptive per-sequence vs per-document selector is driven
by measured kernel latency (`PAPER.md:425-429`: profile the attention kernel
over query/KV lengths, pick the strategy with the lower predicted latency).
The reference expresses that model as a `balsim.profile.v1` CostProfile
(`workload.py:108-193`): a query range of length q attending kv keys costs

    op_scale * padded(q) * kv / throughput(q),  padded(q) = ceil(q / tile) * tile

with `throughput` a piecewise-constant curve on the unpadded q.  This module
times THIS repo's tcgen05 forward + backward kernels on single-range
workloads (q query rows at the end of a kv-token document, the shape every
canonical range has) and fits that exact form, so the same GPU selector
(`wlb_shard_plan`) runs unchanged with the calibrated profile:

    tile_size  = 128 (the kernels' query-tile height)
    op_scale   = 1.0 (latency in seconds)
    throughput = median over kv of padded(q) * kv / measured_seconds, per q bucket

    python -m paper_2503_17924_b200.calibrate --hq 32 --hkv 32 --d 128 --out profile.json
"""

from __future__ import annotations

import argparse
import json
import statistics

import torch

from . import _native
from .attention import attn_backward, attn_forward, build_tiles
from .workload import CostProfile

Q_GRID = (1, 16, 64, 128, 256, 512, 1024, 2048, 4096, 8192)
KV_GRID = (2048, 8192, 32768)


def _time_range(q_len, kv_len, hq, hkv, d, iters, warmup, dev, copies=None):
    """Seconds per range for fwd+bwd of `copies` identical ranges in one launch:
    rows at positions [kv-q, kv) of `copies` documents of kv tokens.

    A rank's ranges all run in one launch, spread over the SMs, so the
    marginal cost of a range in a full-GPU batch (not the latency of a lone
    range, which is launch- and occupancy-bound for small q) is what the
    additive reference model (`sharding.py:151-160`) should be fitted to."""
    if copies is None:
        copies = max(1, min(64, (1 << 17) // kv_len))
    pos = torch.arange(kv_len - q_len, kv_len, dtype=torch.int32, device=dev).repeat(copies)
    rowset = torch.arange(0, (copies + 1) * q_len, q_len, dtype=torch.int32, device=dev)
    tiles = build_tiles(rowset, pos, [kv_len] * copies)
    q = torch.randn(q_len * copies, hq, d, device=dev, dtype=torch.bfloat16)
    k = torch.randn(kv_len * copies, hkv, d, device=dev, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    do = torch.randn_like(q)
    for _ in range(warmup):
        o, lse = attn_forward(q, k, v, tiles)
        attn_backward(q, k, v, o, lse, do, tiles)
    times = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        o, lse = attn_forward(q, k, v, tiles)
        attn_backward(q, k, v, o, lse, do, tiles)
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    return statistics.median(times) / copies


def measure(hq=32, hkv=32, d=128, q_grid=Q_GRID, kv_grid=KV_GRID, iters=5, warmup=2):
    """Latency table {(q, kv): seconds} of the fwd+bwd kernels on this GPU."""
    _native.require_device()
    dev = torch.device("cuda", torch.cuda.current_device())
    table = {}
    for q in q_grid:
        for kv in kv_grid:
            if q <= kv:
                table[(q, kv)] = _time_range(q, kv, hq, hkv, d, iters, warmup, dev)
    return table


def fit_profile(table, tile=128, base: CostProfile | None = None) -> CostProfile:
    """Fit op_scale=1, tile, piecewise-constant throughput(q) to a latency table."""
    base = CostProfile() if base is None else base
    by_q = {}
    for (q, kv), sec in table.items():
        padded = -(-q // tile) * tile
        by_q.setdefault(q, []).append(padded * kv / sec)
    qs = sorted(by_q)
    curve = [(0 if i == 0 else q, statistics.median(by_q[q])) for i, q in enumerate(qs)]
    peak = max(v for _, v in curve)
    return CostProfile(attn_coeff=base.attn_coeff, linear_coeff=base.linear_coeff,
                       linear_const=base.linear_const, tile_size=tile,
                       tflops_curve=tuple(curve), peak_throughput=peak, op_scale=1.0,
                       backward_ratio=base.backward_ratio)


def calibrate(hq=32, hkv=32, d=128, **kw) -> tuple[CostProfile, dict]:
    table = measure(hq, hkv, d, **kw)
    return fit_profile(table), table


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=32)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    profile, table = calibrate(args.hq, args.hkv, args.d)
    profile.to_file(args.out)
    with open(args.out + ".table.json", "w") as fh:
        json.dump({"shape": [args.hq, args.hkv, args.d], "gpu": torch.cuda.get_device_name(),
                   "seconds": {f"{q},{kv}": s for (q, kv), s in sorted(table.items())}},
                  fh, indent=1)
    print(json.dumps(profile.to_dict()))


if __name__ == "__main__":
    main()
