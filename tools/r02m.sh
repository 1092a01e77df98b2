#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/r02m_n$N; mkdir -p $out
timeout 900 python tools/copy_floor.py 32 32 > $out/floor.txt 2>&1; tail -3 $out/floor.txt
for m in auto 4; do
WLB_E2E_GROUPS=$m timeout 500 python bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline > $out/b_$m.json 2> $out/b.err
python -c "
import json
d=json.loads(open('$out/b_$m.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$m', d['value'], e['value'], e['ms_per_step'], e['granularity'], e['rank0_step_ms'])"
done
