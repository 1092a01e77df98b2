#!/usr/bin/env bash
# Multi-micro-batch CP bench vs exchange head groups (WLB_HEAD_GROUPS) and
# pipeline slots, N GPUs, 7B shape, device-side value only.
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/grp_n$N; mkdir -p $out
for rep in 1 2; do
for G in 2 4 8; do
  WLB_HEAD_GROUPS=$G timeout 400 python bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $out/g${G}_$rep.json 2> $out/g${G}_$rep.err
  python -c "
import json; d=json.loads(open('$out/g${G}_$rep.json').read().strip().splitlines()[-1]); print('G=$G rep $rep', d['value'], d.get('imbalance'), d['ms_per_step'])"
done
done
