#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02z
for rep in 1 2; do for o in johnson given; do for G in 4 2; do
WLB_E2E_ORDER=$o WLB_E2E_GROUPS=$G timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --clock-ms 0 > gpurun_out/r02z/b_${o}_${G}_$rep.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/r02z/b_${o}_${G}_$rep.json').read().strip().splitlines()[-1]);print('$o G=$G rep $rep',d['value'],d['e2e']['value'],d['e2e']['ms_per_step'])"
done; done; done 2>&1 | tee gpurun_out/r02z/summary.txt
