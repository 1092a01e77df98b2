#!/usr/bin/env bash
# Multi-GPU round trip (gpurun --gpus N): CP parity worker, single-micro-batch
# overlap probe, bench at N with head groups 4 (default) and 1, GQA shape.
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/${1:-multi}_n$N; mkdir -p $out
timeout 900 python -m pytest tests/test_cp_multi.py -m gpu -q > $out/cp_tests.txt 2>&1; echo "rc=$?" >> $out/cp_tests.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29711 tools/overlap_probe.py > $out/overlap.json 2> $out/overlap.err
timeout 400 python bench.py --gpus $N --steps 5 --warmup 3 > $out/bench.json 2> $out/bench.err
WLB_HEAD_GROUPS=1 timeout 400 python bench.py --gpus $N --steps 5 --warmup 3 --no-e2e > $out/bench_g1.json 2> $out/bench_g1.err
timeout 400 python bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --shape llama70b-gqa > $out/bench_gqa.json 2> $out/bench_gqa.err
tail -3 $out/cp_tests.txt; cat $out/overlap.json; tail -3 $out/overlap.err
for f in bench bench_g1 bench_gqa; do python -c "
import json,sys
try:
    d=json.loads(open('$out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['tflops_per_gpu'], d['imbalance'], d.get('e2e') and d['e2e']['value'], d['config']['strategies'])
except Exception as e: print('$f failed', e); print(open('$out/$f.err').read()[-2000:])
"; done
