"""Re-fit the tile model from the rows of an earlier calibration run (no GPU):
reads tools/calibrate_tiles.py output, fits `calibrate.fit_tile_model`,
re-scores the selection (the other selectors' picks are carried over) and
writes the same report layout and the model file.

    python tools/refit_tiles.py IN.json --hq 32 --hkv 32 --out OUT.json --model-out MODEL.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17924_b200 import calibrate as cal  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("inp")
    ap.add_argument("--hq", type=int, required=True)
    ap.add_argument("--hkv", type=int, required=True)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--out", required=True)
    ap.add_argument("--model-out", default=None)
    a = ap.parse_args()
    old = json.load(open(a.inp))
    rows = old["rows"]
    model = cal.fit_tile_model(rows, a.hq, a.hkv, a.d, device_name=old.get("gpu", "NVIDIA B200"))
    prev = {(r["tag"], r["cp"], r["mb"]): r for r in old["selection"]}
    rep = cal.selection_report(rows, model, {k: v["profile_choice"] for k, v in prev.items()})
    for r in rep:
        p = prev[(r["tag"], r["cp"], r["mb"])]
        r["calibrated_profile_choice"] = p.get("calibrated_profile_choice")
        r["calibrated_profile_correct"] = p.get("calibrated_profile_correct")
    errs = [abs(model.predict(r["features"], r["tl"], r["n_docs"]) * 1e3 / (r["fwd_ms"] + r["bwd_ms"]) - 1)
            for r in rows]
    summ = {}
    for key in sorted({(r["tag"], r["cp"]) for r in rep}):
        rs = [r for r in rep if (r["tag"], r["cp"]) == key]
        summ[f"{key[0]} cp={key[1]}"] = {
            "n": len(rs), "ties": sum(r["tie"] for r in rs),
            "tile_model_correct": sum(r["model_correct"] for r in rs),
            "reference_profile_correct": sum(r["profile_correct"] for r in rs),
            "calibrated_profile_correct": sum(bool(r["calibrated_profile_correct"]) for r in rs),
            "worst_loss_tile_model": round(max(r["loss_if_wrong"] for r in rs), 4)}
    res = dict(old, model=model.to_dict(),
               fit_rel_err={"median": sorted(errs)[len(errs) // 2], "max": max(errs)},
               summary=summ, selection=rep, refit_from=os.path.basename(a.inp))
    tot = {k: sum(v[k] for v in summ.values()) for k in
           ("n", "tile_model_correct", "reference_profile_correct", "calibrated_profile_correct")}
    print(json.dumps({"model": model.to_dict(), "fit_rel_err": res["fit_rel_err"], "totals": tot,
                      "worst": max(v["worst_loss_tile_model"] for v in summ.values())}, indent=1))
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1, default=str)
    if a.model_out:
        model.to_file(a.model_out)


if __name__ == "__main__":
    main()
