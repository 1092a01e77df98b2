#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02w
timeout 300 python tools/copy_floor.py 32 32 2>&1 | tee gpurun_out/r02w/floor.txt
timeout 300 python tools/copy_floor.py 64 8 2>&1 | tee -a gpurun_out/r02w/floor.txt
timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q 2>&1 | tail -3 | tee gpurun_out/r02w/pipe.txt
for G in 4 8; do
WLB_E2E_GROUPS=$G timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --clock-ms 0 > gpurun_out/r02w/b7_$G.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/r02w/b7_$G.json').read().strip().splitlines()[-1]);print('G=$G',d['value'],d['e2e']['value'],d['e2e']['ms_per_step'])"
done
