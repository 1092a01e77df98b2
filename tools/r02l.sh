#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/r02l; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_exchange.py -q -x > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
tail -3 $out/tests.txt
