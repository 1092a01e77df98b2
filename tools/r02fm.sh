#!/usr/bin/env bash
# Final multi-GPU round trip: CP tests, bench (7B, GQA) at N
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/finalm9_n$N; mkdir -p $out
timeout 900 python -m pytest tests/test_cp_multi.py tests/test_gpu_attention.py -k "cp or switches" -m gpu -q > $out/cp_tests.txt 2>&1; echo "rc=$?" >> $out/cp_tests.txt
timeout 700 python bench.py --gpus $N --steps 5 --warmup 3 > $out/bench.json 2> $out/bench.err
timeout 700 python bench.py --gpus $N --steps 5 --warmup 3 --shape llama70b-gqa > $out/bench_gqa.json 2> $out/bench_gqa.err
tail -2 $out/cp_tests.txt
for f in bench bench_gqa; do python -c "
import json
d=json.loads(open('$out/$f.json').read().strip().splitlines()[-1]); e=d.get('e2e') or {}; print('$f', d['value'], d['imbalance'], e.get('value'), e.get('ms_per_step'), (d.get('clocks') or {}).get('reasons'))"; done
