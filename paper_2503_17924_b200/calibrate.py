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


# ------------------------------------------------------------------------------
# Tile model (tilemodel.py): the production measured-latency selector.
# ------------------------------------------------------------------------------

def _time_ms(fn, reps):
    fn()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def measure_tile_workloads(workloads, hq, hkv, d, reps=2, model=None):
    """Per (workload, strategy, rank): the planner's work-list features and the
    MEASURED forward and backward kernel times on this GPU.

    `workloads`: list of (tag, cp, [lengths per micro-batch]).  Each rank's
    kernels run with the full document-ordered K/V resident (exact per-rank
    kernel time; the exchange is not timed)."""
    from .sharding import build_shard_plan
    from .tilemodel import FEATURES, TileModel
    _native.require_device()
    dev = torch.device("cuda", torch.cuda.current_device())
    model = TileModel(hq=hq, hkv=hkv, d=d) if model is None else model
    rows = []
    for tag, cp, mbs in workloads:
        t_max = max(sum(x) for x in mbs)
        q_full = torch.randn(t_max, hq, d, device=dev, dtype=torch.bfloat16)
        k = torch.randn(t_max, hkv, d, device=dev, dtype=torch.bfloat16)
        v = torch.randn_like(k)
        for strat in ("per_sequence", "per_document"):
            plan = build_shard_plan(mbs, cp, strat, model=model)
            feats = plan.features.cpu()
            s_idx = 0 if strat == "per_sequence" else 1
            for b, lengths in enumerate(mbs):
                T = sum(lengths)
                for r in range(cp):
                    g, pos, ro = plan.rank_local(b, r)
                    q = q_full[g.long()]
                    tiles = build_tiles(ro, pos, lengths)
                    kk, vv = k[:T], v[:T]
                    box = {}

                    def fwd():
                        box["o"], box["lse"] = attn_forward(q, kk, vv, tiles)

                    t_f = _time_ms(fwd, reps)
                    # as the CP pipeline runs it: covered dK/dV partial rows
                    # only (the symmetric exchange's covered pull; zero-filling
                    # the rest made per-sequence ranks of short documents look
                    # up to 25 % slower than they run)
                    t_b = _time_ms(lambda: attn_backward(q, kk, vv, box["o"], box["lse"], q, tiles,
                                                         covered_only=cp > 1), reps)
                    rows.append({"tag": tag, "cp": cp, "mb": b, "strategy": strat, "rank": r,
                                 "tl": T // cp, "n_docs": len(lengths),
                                 "features": dict(zip(FEATURES, feats[b, s_idx, r].tolist())),
                                 "fwd_ms": t_f, "bwd_ms": t_b})
        del q_full, k, v
    return rows


def fit_tile_model(rows, hq, hkv, d, sms=148, v3_min_rows=1, device_name=None):
    """Least-squares fit of the tile model to measured rows, forward and
    backward separately, relative residuals (every workload weighs the same
    whatever its size): non-negative per-unit costs, tail weights in [0, 1].
    The costs of the pre-tail linear form (NNLS) seed the non-linear fit."""
    import numpy as np
    from scipy.optimize import least_squares, nnls
    from .tilemodel import TileModel
    f = {k: np.array([r["features"][k] for r in rows], dtype=float)
         for k in rows[0]["features"]}
    v3 = np.array([d == 128 and r["tl"] >= v3_min_rows * max(1, r["n_docs"]) for r in rows])
    yf = np.array([r["fwd_ms"] for r in rows]) * 1e-3
    yb = np.array([r["bwd_ms"] for r in rows]) * 1e-3
    bq = np.where(v3, f["bwd_q128"], f["bwd_q64"])
    bm = np.where(v3, f["bwd_max128"], f["bwd_max64"])

    def t_fwd(x):                       # x = fi, fs, gf, c
        s = (x[0] * f["fwd_items"] + x[1] * f["fwd_steps"]) * hq / sms
        m = x[0] + x[1] * f["fwd_max"]
        return np.maximum(s, m) + x[2] * np.minimum(s, m) + x[3]

    def t_bwd(x):                       # x = bi64, bi128, bs64, bs128, gb, c
        # per-item costs split by kernel: the persistent 64-query kernel's
        # items are far cheaper than the 128-query kernel's
        bi = np.where(v3, x[1], x[0])
        bs = np.where(v3, x[3], x[2])
        s = (bi * f["bwd_items"] * hkv + bs * bq * hq) / sms
        m = bi + bs * bm * hq / hkv
        return np.maximum(s, m) + x[4] * np.minimum(s, m) + x[5]

    def seed(cols, y):
        a = np.stack(cols, 1) / y[:, None]
        return nnls(a, np.ones_like(y))[0]

    sf = seed([f["fwd_items"] * hq / sms, f["fwd_steps"] * hq / sms, np.ones_like(yf)], yf)
    items = f["bwd_items"] * hkv / sms
    sb = seed([np.where(v3, 0, items), np.where(v3, items, 0), np.where(v3, 0, bq * hq / sms),
               np.where(v3, bq * hq / sms, 0), np.ones_like(yb)], yb)
    inf = np.inf
    xf = least_squares(lambda x: t_fwd(x) / yf - 1, [sf[0], sf[1], 0.0, sf[2]],
                       bounds=([0, 0, 0, 0], [inf, inf, 1, inf]), x_scale="jac").x
    # a kernel no row ran keeps its seed costs (no data moves them)
    xb = np.array([*sb[:4], 0.0, sb[4]])
    act = [i for i in range(6) if not ((i in (0, 2) and v3.all()) or (i in (1, 3) and not v3.any()))]

    def rb(x):
        xb[act] = x
        return t_bwd(xb) / yb - 1

    hi = np.array([inf, inf, inf, inf, 1, inf])[act]
    xb[act] = least_squares(rb, xb[act], bounds=(np.zeros(len(act)), hi), x_scale="jac").x
    return TileModel(hq=hq, hkv=hkv, d=d, sms=sms, fwd_item_s=float(xf[0]),
                     fwd_step_s=float(xf[1]), bwd_item_s=float(xb[0]), bwd_item128_s=float(xb[1]),
                     bwd_step64_s=float(xb[2]), bwd_step128_s=float(xb[3]),
                     v3_min_rows=v3_min_rows, const_s=float(xf[3] + xb[5]),
                     fwd_tail=float(xf[2]), bwd_tail=float(xb[4]),
                     source=f"least squares over {len(rows)} measured rank workloads on "
                            f"{device_name or torch.cuda.get_device_name()}")


def selection_report(rows, model, profile_choices=None):
    """Per (workload, micro-batch): measured group time of each strategy (max
    over ranks of fwd + bwd), the measured-faster strategy, the tile model's
    choice and (optionally) another selector's choices keyed like the rows.
    Identical shardings (e.g. a single document) are ties: any choice is right."""
    groups = {}
    for r in rows:
        key = (r["tag"], r["cp"], r["mb"])
        g = groups.setdefault(key, {"per_sequence": [], "per_document": []})
        g[r["strategy"]].append(r)
    out = []
    for key, g in sorted(groups.items()):
        meas = {s: max(x["fwd_ms"] + x["bwd_ms"] for x in g[s]) for s in g}
        pred = {s: max(model.predict(x["features"], x["tl"], x["n_docs"]) for x in g[s])
                for s in g}
        same = [x["features"] for x in g["per_sequence"]] == [x["features"] for x in g["per_document"]]
        best = min(meas, key=meas.get)
        pick = "per_sequence" if pred["per_sequence"] <= pred["per_document"] else "per_document"
        rec = {"tag": key[0], "cp": key[1], "mb": key[2], "measured_ms": meas,
               "predicted_ms": {s: v * 1e3 for s, v in pred.items()}, "measured_best": best,
               "model_choice": pick, "tie": same,
               "model_correct": same or pick == best,
               "loss_if_wrong": 0.0 if same or pick == best else meas[pick] / meas[best] - 1}
        if profile_choices is not None:
            c = profile_choices.get(key)
            rec["profile_choice"] = c
            rec["profile_correct"] = same or c == best
        out.append(rec)
    return out


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
