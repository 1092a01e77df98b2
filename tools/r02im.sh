#!/usr/bin/env bash
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out/im
for c in 100 0 100 0; do
timeout 600 python bench.py --gpus $N --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --clock-ms $c > gpurun_out/im/b.json 2> gpurun_out/im/b.err
python -c "
import json
d=json.loads(open('gpurun_out/im/b.json').read().strip().splitlines()[-1]); print('clock-ms $c', d['value'], d['imbalance'], d['rank_kernel_ms'])"
done
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,pcie.link.gen.current --format=csv
