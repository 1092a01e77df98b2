"""Calibrate the measured-latency CP selector (tilemodel.TileModel) on B200
and report how well it picks the faster strategy.

Workloads: the 8 synthetic 32K and 128K sequences of bench.py at cp = 1..8,
plus a sample of BASELINE config 5 micro-batches (W(d) packer with outlier
queues, padded for CP=8).  For every (micro-batch, strategy, rank) the
planner's work-list features and the measured forward / backward kernel
times are recorded; the model's five per-unit costs are fitted by least
squares; then, per micro-batch, the measured-faster strategy is compared
with the choices of (a) the tile model, (b) the reference CostProfile
(bit-exact balsim selector) and (c) the reference-form profile calibrated by
`calibrate.py` (round 1).

    python tools/calibrate_tiles.py --hq 32 --hkv 32 --out profiles/r02_tiles_7b.json \
        --model-out paper_2503_17924_b200/data/b200_tiles_h32_kv32_d128.json
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_17924_b200 as wl  # noqa: E402
from paper_2503_17924_b200 import calibrate as cal  # noqa: E402


def synthetic(window, n=8):
    spec = wl.SyntheticSpec(context_window=window, tokens_per_global_batch=window)
    return [[d.length for d in b] for b in wl.generate_synthetic_stream(spec, 0, n)]


def config5(iters, sample, cp=8):
    """Micro-batches of config 5 (heaviest and lightest of each iteration)."""
    prof = wl.CostProfile()
    spec = wl.SyntheticSpec(context_window=131072, tokens_per_global_batch=64 * 131072)
    packer = wl.HeuristicPacker(wl.OutlierQueueSet((32768, 98304)), 64, 163840, prof)
    filler = wl._FillerIds()
    out = []
    for it, batch in enumerate(wl.generate_synthetic_stream(spec, 0, iters)):
        plan = packer.feed(batch, it)
        mbs = [wl.pad_for_cp(mb, cp, filler, it).lengths() for mb in plan.microbatches if mb.docs]
        mbs.sort(key=lambda ls: -sum(x * (x + 1) // 2 for x in ls))
        pick = mbs[:sample // 2] + mbs[-(sample - sample // 2):]
        out.append((f"config5-it{it}", cp, pick))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=32)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--c5-iters", type=int, default=2)
    ap.add_argument("--c5-sample", type=int, default=8)
    ap.add_argument("--quick", action="store_true", help="fewer workloads (smoke)")
    ap.add_argument("--out", required=True)
    ap.add_argument("--model-out", default=None)
    a = ap.parse_args()
    seq32, seq128 = synthetic(32768), synthetic(131072)
    pad = lambda ls, cp: wl.pad_for_cp(wl.MicroBatch([wl.Document(i, x) for i, x in enumerate(ls)]),
                                       cp, wl._FillerIds(), 0).lengths()
    cps32, cps128 = ((1, 2, 4, 8), (2, 4, 8)) if not a.quick else ((2,), (8,))
    work = [(f"32k", cp, [pad(x, cp) for x in seq32]) for cp in cps32]
    work += [(f"128k", cp, [pad(x, cp) for x in seq128]) for cp in cps128]
    work += config5(a.c5_iters if not a.quick else 1, a.c5_sample if not a.quick else 2)
    rows = cal.measure_tile_workloads(work, a.hq, a.hkv, a.d, reps=a.reps)
    model = cal.fit_tile_model(rows, a.hq, a.hkv, a.d)
    # other selectors' choices on the same micro-batches
    ref_choice, prof_choice = {}, {}
    prof_path = os.path.join(os.path.dirname(wl.__file__), "data",
                             "b200_llama7b_h32_d128.profile.json" if a.hq == 32 else
                             "b200_llama70b_h64_kv8_d128.profile.json")
    cal_prof = wl.CostProfile.from_file(prof_path) if os.path.exists(prof_path) else None
    for tag, cp, mbs in work:
        rp = wl.build_shard_plan(mbs, cp, "adaptive", wl.CostProfile(), with_tokens=False)
        cpn = wl.build_shard_plan(mbs, cp, "adaptive", cal_prof, with_tokens=False) if cal_prof else None
        for b in range(len(mbs)):
            ref_choice[(tag, cp, b)] = rp.strategy(b).value
            if cpn is not None:
                prof_choice[(tag, cp, b)] = cpn.strategy(b).value
    rep = cal.selection_report(rows, model, ref_choice)
    for r in rep:
        r["calibrated_profile_choice"] = prof_choice.get((r["tag"], r["cp"], r["mb"]))
        r["calibrated_profile_correct"] = r["tie"] or r["calibrated_profile_choice"] == r["measured_best"]
    # fit quality
    errs = [abs(model.predict(r["features"], r["tl"], r["n_docs"]) * 1e3 / (r["fwd_ms"] + r["bwd_ms"]) - 1)
            for r in rows]
    summ = {}
    for key in sorted({(r["tag"], r["cp"]) for r in rep}):
        rs = [r for r in rep if (r["tag"], r["cp"]) == key]
        summ[f"{key[0]} cp={key[1]}"] = {
            "n": len(rs), "ties": sum(r["tie"] for r in rs),
            "tile_model_correct": sum(r["model_correct"] for r in rs),
            "reference_profile_correct": sum(r["profile_correct"] for r in rs),
            "calibrated_profile_correct": sum(r["calibrated_profile_correct"] for r in rs),
            "worst_loss_tile_model": round(max(r["loss_if_wrong"] for r in rs), 4)}
    res = {"shape": [a.hq, a.hkv, a.d], "gpu": torch.cuda.get_device_name(),
           "model": model.to_dict(),
           "fit_rel_err": {"median": sorted(errs)[len(errs) // 2], "max": max(errs)},
           "summary": summ, "selection": rep, "rows": rows}
    print(json.dumps({"model": model.to_dict(), "fit_rel_err": res["fit_rel_err"],
                      "summary": summ}, indent=1), flush=True)
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1, default=str)
    if a.model_out:
        model.to_file(a.model_out)


if __name__ == "__main__":
    main()
