#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for o in johnson given; do ORDER=$o timeout 300 python tools/e2e_timeline.py 4; done 2>&1 | tee gpurun_out/e2e_timeline.txt
timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q 2>&1 | tail -2
for s in llama7b llama70b-gqa; do
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --clock-ms 0 --shape $s > gpurun_out/b_$s.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/b_$s.json').read().strip().splitlines()[-1]);print('$s',d['value'],d['e2e']['value'],d['e2e']['ms_per_step'])"
done
