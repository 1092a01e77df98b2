#!/usr/bin/env bash
# Tile model with list-scheduling tail terms: GPU selector tests, whole GPU
# suite, smoke, config 5 under the re-fitted model.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/tail; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_tests.txt 2>&1; echo "all rc=$?" >> $out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "smoke rc=$?" >> $out/smoke.txt
timeout 900 python tools/config5.py --out $out/config5.jsonl > $out/config5.txt 2>&1
tail -n 2 $out/gpu_tests.txt; tail -n 1 $out/smoke.txt; tail -n 4 $out/config5.txt | cut -c1-300
