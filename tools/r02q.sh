#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/r02q; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_exchange.py -q -x > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
tail -2 $out/tests.txt
bash tools/ab_run.sh ab7 G2 K
