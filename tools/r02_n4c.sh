#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/n4c_n$N; mkdir -p $out
for mode in covered dma; do
  for s in 0 2; do
    WLB_XCHG_PUSH=$mode timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2972$s tools/overlap_probe.py --seq $s --groups 1 4 > $out/overlap_${mode}_s$s.json 2> $out/overlap_${mode}_s$s.err
    echo "$mode seq $s"; cat $out/overlap_${mode}_s$s.json | cut -c1-600; tail -2 $out/overlap_${mode}_s$s.err
  done
  WLB_XCHG_PUSH=$mode timeout 400 python bench.py --gpus $N --steps 5 --warmup 3 --no-e2e > $out/bench_$mode.json 2> $out/bench_$mode.err
  python -c "
import json
d=json.loads(open('$out/bench_$mode.json').read().strip().splitlines()[-1]); print('$mode bench', d['value'], d['imbalance'])" 2>&1 | tail -1
done
