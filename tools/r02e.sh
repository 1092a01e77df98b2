#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/r02e; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_exchange.py tests/test_gpu_scale.py -q -x > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
for p in 0 1; do timeout 300 python tools/short_profile.py --bwd-persistent $p > $out/short_p$p.jsonl 2>&1; done
for p in 0 1; do timeout 600 python tools/config5.py --iters 2 --sample 8 --bwd-persistent $p --out $out/config5_p$p.json > $out/config5_p$p.log 2>&1; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $out/bench_n1.json 2>&1
tail -2 $out/tests.txt
