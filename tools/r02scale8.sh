#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/scale8; mkdir -p $out; rm -f $out/parity.jsonl
WLB_PARITY_LOG=$out/parity.jsonl timeout 900 python -m pytest tests/test_gpu_scale.py -k "cp8" -m gpu -q > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
tail -2 $out/tests.txt; cut -c1-300 $out/parity.jsonl
