"""Leave-one-workload-out check of the tile model (no GPU): for every
(workload, cp) group of a calibration run, fit `calibrate.fit_tile_model` on
the other groups' rows and score the held-out group's strategy picks.

    python tools/cv_tiles.py profiles/r02_tile_model_calibration_llama70b_gqa.json --hq 64 --hkv 8
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
    a = ap.parse_args()
    rows = json.load(open(a.inp))["rows"]
    groups = sorted({(r["tag"], r["cp"]) for r in rows})
    ok = n = 0
    worst = 0.0
    for g in groups:
        train = [r for r in rows if (r["tag"], r["cp"]) != g]
        test = [r for r in rows if (r["tag"], r["cp"]) == g]
        m = cal.fit_tile_model(train, a.hq, a.hkv, a.d, device_name="held-out fit")
        rep = cal.selection_report(test, m)
        good = sum(r["model_correct"] for r in rep)
        ok += good
        n += len(rep)
        worst = max([worst] + [r["loss_if_wrong"] for r in rep])
        print(f"{g[0]} cp={g[1]}: {good}/{len(rep)} (tails {m.fwd_tail:.2f}/{m.bwd_tail:.2f})")
    print(json.dumps({"held_out_correct": ok, "n": n, "worst_loss": round(worst, 4)}))


if __name__ == "__main__":
    main()
