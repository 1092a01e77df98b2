#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02z
for rep in 1 2 3; do for G in auto mb; do for s in llama7b; do
WLB_E2E_GROUPS=$G timeout 400 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --clock-ms 0 --shape $s > gpurun_out/r02z/b.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/r02z/b.json').read().strip().splitlines()[-1]);e=d['e2e'];print('$s G=$G rep $rep',d['value'],e['value'],e['ms_per_step'],e['granularity'],e['rank0_step_ms'])"
done; done; done 2>&1 | tee gpurun_out/r02z/summary.txt
