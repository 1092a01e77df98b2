"""Score a tile model (no fit) on the rows of a calibration run: strategy
picks vs the measured-faster strategy per micro-batch, and the prediction's
relative error.  Used to check the shipped models on fresh measurements.

    python tools/score_tiles.py ROWS.json [--model paper_2503_17924_b200/data/b200_tiles_h32_kv32_d128.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_17924_b200 import calibrate as cal  # noqa: E402
from paper_2503_17924_b200.tilemodel import TileModel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rows")
    ap.add_argument("--model", default=None, help="model file (default: shipped for the shape)")
    a = ap.parse_args()
    d = json.load(open(a.rows))
    hq, hkv, hd = d["shape"]
    m = TileModel.from_file(a.model) if a.model else TileModel.for_shape(hq, hkv, hd)
    rep = cal.selection_report(d["rows"], m)
    errs = sorted(abs(m.predict(r["features"], r["tl"], r["n_docs"]) * 1e3 / (r["fwd_ms"] + r["bwd_ms"]) - 1)
                  for r in d["rows"])
    out = {"rows": os.path.basename(a.rows), "model": m.source, "tails": [m.fwd_tail, m.bwd_tail],
           "correct": sum(r["model_correct"] for r in rep), "n": len(rep),
           "worst_loss": round(max(r["loss_if_wrong"] for r in rep), 4),
           "rel_err_median": round(errs[len(errs) // 2], 4), "rel_err_max": round(errs[-1], 4),
           "misses": [(r["tag"], r["cp"], r["mb"], round(r["loss_if_wrong"], 4)) for r in rep
                      if not r["model_correct"]]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
