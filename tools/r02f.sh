#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/r02f; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_attention.py -q -x > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
tail -3 $out/tests.txt
bash tools/ab_run.sh ab3 A B E F
