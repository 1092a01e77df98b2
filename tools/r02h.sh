#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/r02h; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -k "project or fused" > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
tail -30 $out/tests.txt
timeout 300 python tools/proj_bench.py > $out/proj_bench.jsonl 2>&1
cat $out/proj_bench.jsonl
