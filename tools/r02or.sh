#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/or
for rep in 1 2; do for s in llama70b-gqa llama7b; do for o in given johnson; do
WLB_E2E_ORDER=$o timeout 400 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --clock-ms 0 --shape $s > gpurun_out/or/b.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/or/b.json').read().strip().splitlines()[-1]);e=d['e2e'];print('$s $o rep $rep',d['value'],e['value'],e['ms_per_step'],e['order'])"
done; done; done 2>&1 | tee gpurun_out/or/summary.txt
