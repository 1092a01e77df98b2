#!/usr/bin/env bash
# Same-box A/B of library builds in var/lib<name>.so: tools/ab_run.sh <out> A B C ...
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/$1; shift
mkdir -p $out
for rep in 1 2; do
  for n in "$@"; do
    export WLB_LIB_PATH=var/lib$n.so
    timeout 300 python tools/short_profile.py --ranks 4 > $out/short_${n}_$rep.jsonl 2>&1
    timeout 600 python tools/config5.py --iters 2 --sample 4 --out $out/c5_${n}_$rep.json > /dev/null 2>&1
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --clock-ms 0 > $out/bench_${n}_$rep.json 2>&1
  done
done
unset WLB_LIB_PATH
python - "$out" "$@" <<'PY'
import json, sys
out, names = sys.argv[1], sys.argv[2:]
for n in names:
    for rep in (1, 2):
        try:
            sp = [json.loads(l) for l in open(f"{out}/short_{n}_{rep}.jsonl")]
            c5 = json.load(open(f"{out}/c5_{n}_{rep}.json"))
            b = json.load(open(f"{out}/bench_{n}_{rep}.json"))
        except Exception as e:
            print(n, rep, "failed", e); continue
        print(n, rep, "short", [(r["strategy"][4:7], r["tflops_per_gpu"]) for r in sp],
              "c5", [round(sum(s["tflops_per_gpu"] for s in it["sample"]) / len(it["sample"]), 1) for it in c5],
              "bench", b["value"])
PY
