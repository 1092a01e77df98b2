"""Where the time goes on short-document CP ranks (BASELINE config 5).

Takes the config-5 packer's micro-batches (CP=8), and for the lightest and
heaviest micro-batch of iteration 0 times, per rank and strategy, every
launch of the attention path separately with CUDA events: the tile lists,
the forward, and the backward's pieces (run through the public entry
points).  Under ncu (`--metrics gpu__time_duration.sum`) the same run gives
the per-kernel launch list.

    python tools/short_profile.py [--mb 0] [--cp 8] [--ranks 8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.attention import attn_backward, attn_forward, build_tiles  # noqa: E402


def ev_ms(fn, reps=3):
    fn()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cp", type=int, default=8)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--full-partials", action="store_true",
                    help="zero-fill uncovered dK/dV rows (the single-rank API) instead of the "
                         "CP pipeline's covered-only backward")
    ap.add_argument("--bwd-persistent", type=int, default=-1)
    ap.add_argument("--v3-min-rows", type=int, default=-1,
                    help="backward kernel threshold override (0: always the 128-query kernel)")
    a = ap.parse_args()
    from paper_2503_17924_b200.attention import set_bwd_v3_min_rows
    if a.v3_min_rows >= 0:
        set_bwd_v3_min_rows(a.v3_min_rows)
    from paper_2503_17924_b200.attention import set_bwd_persistent
    if a.bwd_persistent >= 0:
        set_bwd_persistent(a.bwd_persistent)
    dev = torch.device("cuda")
    prof = wl.CostProfile()
    spec = wl.SyntheticSpec(context_window=131072, tokens_per_global_batch=64 * 131072)
    packer = wl.HeuristicPacker(wl.OutlierQueueSet((32768, 98304)), 64, 163840, prof)
    batch = wl.generate_synthetic_stream(spec, 0, 1)[0]
    plan_h = packer.feed(batch, 0)
    mbs = [wl.pad_for_cp(mb, a.cp, wl._FillerIds(), 0).lengths()
           for mb in plan_h.microbatches if mb.docs]
    mbs.sort(key=lambda ls: sum(x * (x + 1) // 2 for x in ls))
    d = 128
    for name, lengths in (("lightest", mbs[0]), ("heaviest", mbs[-1])):
        T = sum(lengths)
        q_full = torch.randn(T, a.hq, d, device=dev, dtype=torch.bfloat16)
        k = torch.randn(T, a.hkv, d, device=dev, dtype=torch.bfloat16)
        v = torch.randn_like(k)
        pairs = sum(x * (x + 1) // 2 for x in lengths)
        for strat in ("per_sequence", "per_document"):
            plan = wl.build_shard_plan([lengths], a.cp, strat)
            rec = {"mb": name, "tokens": T, "docs": len(lengths), "strategy": strat, "ranks": []}
            for r in range(min(a.ranks, a.cp)):
                g, pos, ro = plan.rank_local(0, r)
                q = q_full[g.long()]
                box = {}

                def tiles():
                    box["t"] = build_tiles(ro, pos, lengths)

                t_tiles = ev_ms(tiles, a.reps)

                def fwd():
                    box["o"], box["lse"] = attn_forward(q, k, v, box["t"])

                t_fwd = ev_ms(fwd, a.reps)
                t_bwd = ev_ms(lambda: attn_backward(q, k, v, box["o"], box["lse"], q, box["t"],
                                                    covered_only=not a.full_partials), a.reps)
                rp = int(plan.rank_pairs[0, r].item())
                rec["ranks"].append({"rank": r, "rows": q.shape[0], "pairs": rp,
                                     "tiles_ms": round(t_tiles, 4), "fwd_ms": round(t_fwd, 4),
                                     "bwd_ms": round(t_bwd, 4),
                                     "fwd_tflops": round(4 * d * a.hq * rp / t_fwd / 1e9, 1),
                                     "bwd_tflops": round(10 * d * a.hq * rp / t_bwd / 1e9, 1)})
            tot = [x["tiles_ms"] + x["fwd_ms"] + x["bwd_ms"] for x in rec["ranks"]]
            rec["max_rank_ms"] = round(max(tot), 4)
            rec["imbalance"] = round(max(tot) / (sum(tot) / len(tot)), 4)
            rec["tflops_per_gpu"] = round(14 * d * a.hq * pairs / a.cp / max(tot) / 1e9, 1)
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
