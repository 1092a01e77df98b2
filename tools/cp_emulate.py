"""Emulate CP=N ranks on one GPU (hard part 5).

Given the full document-ordered K/V, each CP rank's attention is independent,
so every rank's fwd+bwd kernels can be replayed on one B200 and timed exactly.
For each synthetic sequence and cp, both strategies are measured:

  * per-rank kernel time t_r (CUDA events), group time max_r t_r,
    imbalance max/mean, TFLOP/s per rank-GPU;
  * the measured-faster strategy vs the choice of the reference-model selector
    (default CostProfile, bit-exact with balsim) and of the selector with the
    profile calibrated from measured kernel latency (calibrate.py).

    python tools/cp_emulate.py --window 131072 --cps 4 8 --profile p.json --out r.json
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200.attention import attn_backward, attn_forward, build_tiles  # noqa: E402


def rank_times(plan, b, cp, q_full, k, v, do_full, reps):
    lengths = plan.lengths[b]
    out = []
    for r in range(cp):
        g, pos, ro = plan.rank_local(b, r)
        idx = g.long()
        q, do = q_full[idx], do_full[idx]
        tiles = build_tiles(ro, pos, lengths)
        o, lse = attn_forward(q, k, v, tiles)
        attn_backward(q, k, v, o, lse, do, tiles)
        ts = []
        for _ in range(reps):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            o, lse = attn_forward(q, k, v, tiles)
            attn_backward(q, k, v, o, lse, do, tiles)
            e.record()
            e.synchronize()
            ts.append(a.elapsed_time(e))
        out.append(min(ts))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--window", type=int, default=131072)
    ap.add_argument("--cps", type=int, nargs="+", default=[4, 8])
    ap.add_argument("--seqs", type=int, default=8)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=32)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--profile", default=None)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda")
    spec = wl.SyntheticSpec(args.window, args.window)
    stream = [[d.length for d in b] for b in wl.generate_synthetic_stream(spec, 0, args.seqs)]
    ref_prof = wl.CostProfile()
    cal_prof = wl.CostProfile.from_file(args.profile) if args.profile else None
    T = args.window
    q_full = torch.randn(T, args.hq, args.d, device=dev, dtype=torch.bfloat16)
    k = torch.randn(T, args.hkv, args.d, device=dev, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    do_full = torch.randn_like(q_full)
    rows = []
    for cp in args.cps:
        lengths = [wl.pad_for_cp(wl.MicroBatch([wl.Document(i, x) for i, x in enumerate(ls)]),
                                 cp, wl._FillerIds(), 0).lengths() for ls in stream]
        plans = {s: wl.build_shard_plan(lengths, cp, s) for s in ("per_sequence", "per_document")}
        ref_choice = wl.build_shard_plan(lengths, cp, "adaptive", ref_prof, with_tokens=False)
        cal_choice = (wl.build_shard_plan(lengths, cp, "adaptive", cal_prof, with_tokens=False)
                      if cal_prof else None)
        for b, ls in enumerate(lengths):
            pairs = sum(x * (x + 1) // 2 for x in ls)
            flops = 14.0 * args.d * args.hq * pairs
            rec = {"cp": cp, "seq": b, "docs": len(ls), "max_doc": max(ls)}
            for s, plan in plans.items():
                t = rank_times(plan, b, cp, q_full, k, v, do_full, args.reps)
                mx, mean = max(t), sum(t) / len(t)
                rec[s] = {"rank_ms": [round(x, 3) for x in t], "group_ms": round(mx, 3),
                          "imbalance": round(mx / mean, 4),
                          "tflops_per_gpu": round(flops / cp / (mx / 1e3) / 1e12, 1),
                          "pair_imbalance": round(float(plan.rank_pairs[b].max()) /
                                                  float(plan.rank_pairs[b].double().mean()), 5)}
            best = min(plans, key=lambda s: rec[s]["group_ms"])
            rec["measured_best"] = best
            rec["ref_model_choice"] = ref_choice.strategy(b).value
            if cal_choice is not None:
                rec["calibrated_choice"] = cal_choice.strategy(b).value
            rows.append(rec)
            print(json.dumps(rec), flush=True)
    summ = {}
    for cp in args.cps:
        rs = [r for r in rows if r["cp"] == cp]
        summ[cp] = {
            "ref_model_correct": sum(r["ref_model_choice"] == r["measured_best"] for r in rs),
            "calibrated_correct": (sum(r.get("calibrated_choice") == r["measured_best"] for r in rs)
                                   if cal_prof else None),
            "n": len(rs),
            "mean_imbalance_per_doc": round(sum(r["per_document"]["imbalance"] for r in rs) / len(rs), 4),
            "mean_imbalance_per_seq": round(sum(r["per_sequence"]["imbalance"] for r in rs) / len(rs), 4),
        }
    print(json.dumps({"summary": summ}), flush=True)
    if args.out:
        json.dump({"rows": rows, "summary": summ}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
