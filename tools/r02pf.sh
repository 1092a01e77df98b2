#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/l2pf; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_attention.py -m gpu -q -x > $out/attn_tests.txt 2>&1; echo "rc=$?" >> $out/attn_tests.txt
timeout 600 python tools/l2pf_ab.py > $out/ab_7b.txt 2>&1
timeout 600 python tools/l2pf_ab.py --hq 64 --hkv 8 --reps 3 > $out/ab_gqa.txt 2>&1
tail -2 $out/attn_tests.txt; cat $out/ab_7b.txt; cat $out/ab_gqa.txt
