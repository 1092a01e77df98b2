#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/so; mkdir -p $out
timeout 600 python tools/stream_overlap_probe.py > $out/7b.txt 2>&1; cat $out/7b.txt
timeout 600 python tools/stream_overlap_probe.py --hq 64 --hkv 8 --reps 3 > $out/gqa.txt 2>&1; cat $out/gqa.txt
