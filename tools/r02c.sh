#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/r02c; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_shard.py tests/test_gpu_attention.py -q -x > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
timeout 300 python tools/short_profile.py > $out/short_profile.jsonl 2>&1
timeout 600 python tools/config5.py --iters 2 --sample 8 --out $out/config5.json > $out/config5.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench_n1.json 2>&1
bash tools/sanitize.sh > $out/sanitize_summary.txt 2>&1
tail -2 $out/tests.txt; cat $out/config5.log | cut -c1-400; cat $out/bench_n1.json | cut -c1-300; cat $out/sanitize_summary.txt
