#!/usr/bin/env bash
# Same-box A/B of the round-1 snapshot (var/r01) and the current tree at N GPUs.
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/abm_n$N; mkdir -p $out
for rep in 1 2; do
  # (the round-1 bench.py does not launch torchrun itself)
  (cd var/r01 && timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2960$rep bench.py --gpus $N --steps 5 --warmup 3 --no-e2e > ../../$out/r01_$rep.json 2>/dev/null)
  timeout 900 python bench.py --gpus $N --steps 5 --warmup 3 --no-e2e > $out/cur_$rep.json 2>/dev/null
  WLB_XCHG_DKV=bf16 timeout 900 python bench.py --gpus $N --steps 5 --warmup 3 --no-e2e > $out/curbf16_$rep.json 2>/dev/null
done
for f in $out/*.json; do python -c "
import json
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['imbalance'], d['rank_kernel_ms'], d.get('rank_mb_kernel_ms'))
except Exception as e: print('$f failed', e)
"; done
