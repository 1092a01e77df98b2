#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for G in 4 2; do timeout 300 python tools/e2e_timeline.py $G 64 8; done 2>&1 | tee gpurun_out/e2e_timeline_gqa.txt
timeout 300 python tools/copy_floor.py 64 8 2>&1 | tail -4
