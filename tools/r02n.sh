#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/r02n_n$N; mkdir -p $out
pr() { python -c "
import json
d=json.loads(open('$1').read().strip().splitlines()[-1]); e=d['e2e']; print('$2', d['value'], e['value'], e['ms_per_step'], e.get('rank0_step_ms'))"; }
for rep in 1; do
(cd var/old && timeout 500 python bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline > ../../$out/old.json 2> ../../$out/old.err); pr $out/old.json old
WLB_E2E_ORDER=given WLB_E2E_GROUPS=mb timeout 500 python bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline > $out/new.json 2> $out/new.err; pr $out/new.json mb-given
WLB_E2E_ORDER=given WLB_E2E_GROUPS=4 timeout 500 python bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline > $out/new.json 2> $out/new.err; pr $out/new.json g4-given
done
