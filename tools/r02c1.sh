#!/usr/bin/env bash
# BASELINE config 1 (8K, 8 heads, D=64, CP=2 per-document): parity + CPU
# reference path timed beside the GPU kernels; scheduling-switch test.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/c1; mkdir -p $out; rm -f $out/config1.jsonl
nproc > $out/nproc.txt; lscpu | grep "Model name" >> $out/nproc.txt
WLB_CONFIG1_LOG=$out/config1.jsonl timeout 900 python -m pytest tests/test_gpu_config1.py tests/test_gpu_attention.py -k "config1 or switches" -m gpu -q > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
tail -3 $out/tests.txt; cat $out/nproc.txt; cut -c1-400 $out/config1.jsonl
