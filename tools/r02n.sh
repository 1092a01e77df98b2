#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/r02n_n$N; mkdir -p $out
timeout 240 python -m pytest tests/test_gpu_exchange.py -q -x > $out/tests.txt 2>&1; echo "1gpu tests rc=$? $(tail -1 $out/tests.txt)"
WLB_XCHG_PUSH=dma timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29851 tests/cp_worker.py > $out/worker.log 2>&1; echo "worker rc=$? $(grep -c 'CP OK' $out/worker.log)"
for s in 0 2; do
  WLB_XCHG_PUSH=dma timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2973$s tools/overlap_probe.py --seq $s --groups 1 4 > $out/overlap_dma_s$s.json 2> $out/overlap_dma_s$s.err
  echo "dma seq $s: $(cut -c1-700 $out/overlap_dma_s$s.json) $(grep -m1 -iE 'error' $out/overlap_dma_s$s.err | cut -c1-300)"
done
WLB_XCHG_PUSH=dma timeout 400 python bench.py --gpus $N --steps 5 --warmup 3 --no-e2e > $out/bench_dma.json 2> $out/bench_dma.err
python -c "
import json
d=json.loads(open('$out/bench_dma.json').read().strip().splitlines()[-1]); print('dma bench', d['value'], d['imbalance'])" 2>&1 | tail -1
timeout 400 python bench.py --gpus $N --steps 5 --warmup 3 --no-e2e > $out/bench_cov.json 2> $out/bench_cov.err
python -c "
import json
d=json.loads(open('$out/bench_cov.json').read().strip().splitlines()[-1]); print('covered bench', d['value'], d['imbalance'])" 2>&1 | tail -1
