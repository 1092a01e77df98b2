#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/r02d; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_exchange.py -q -x > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
for p in 0 1; do timeout 300 python tools/short_profile.py --bwd-persistent $p > $out/short_p$p.jsonl 2>&1; done
timeout 600 python tools/config5.py --iters 2 --sample 8 --out $out/config5.json > $out/config5.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $out/bench_n1.json 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --shape llama70b-gqa > $out/bench_n1_gqa.json 2>&1
tail -2 $out/tests.txt; for p in 0 1; do cut -c1-200 $out/short_p$p.jsonl; done; cut -c1-300 $out/config5.log; cut -c1-200 $out/bench_n1*.json
