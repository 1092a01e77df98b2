#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/r02m_n$N; mkdir -p $out
for m in groups mb; do
WLB_E2E_MODE=$m timeout 500 python bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline > $out/b.json 2> $out/b.err
python -c "
import json
d=json.loads(open('$out/b.json').read().strip().splitlines()[-1]); print('$m', d['value'], d['alloc_retries'], d['e2e'])"
done
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True WLB_E2E_MODE=groups timeout 500 python bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline > $out/b.json 2> $out/b.err
python -c "
import json
d=json.loads(open('$out/b.json').read().strip().splitlines()[-1]); print('groups expandable', d['value'], d['alloc_retries'], d['e2e'])"
