#!/usr/bin/env bash
cd "$(dirname "$0")/.."
WLB_LIB_PATH=var/libq1.so timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_scale.py tests/test_gpu_exchange.py -x -q 2>&1 | tail -2
cat > /tmp/cp4.py <<'PY'
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, paper_2503_17924_b200 as wl
from paper_2503_17924_b200 import calibrate as cal
spec = wl.SyntheticSpec(context_window=32768, tokens_per_global_batch=32768)
seqs = [[d.length for d in b] for b in wl.generate_synthetic_stream(spec, 0, 8)]
pad = lambda ls, cp: wl.pad_for_cp(wl.MicroBatch([wl.Document(i, x) for i, x in enumerate(ls)]), cp, wl._FillerIds(), 0).lengths()
for hq, hkv in ((64, 8), (32, 32)):
    for cp in (2, 4):
        rows = cal.measure_tile_workloads([("32k", cp, [pad(x, cp) for x in seqs])], hq, hkv, 128, reps=2)
        g = {}
        for r in rows:
            g.setdefault((r["mb"], r["strategy"]), []).append(r["fwd_ms"] + r["bwd_ms"])
        tot = {s: round(sum(max(v) for (mb, st), v in g.items() if st == s), 3) for s in ("per_sequence", "per_document")}
        print(os.environ.get("TAG"), hq, hkv, cp, tot, flush=True)
PY
for n in q0 q1; do TAG=$n WLB_LIB_PATH=var/lib$n.so timeout 600 python /tmp/cp4.py; done
bash tools/ab_n1.sh qrot q0 q1
