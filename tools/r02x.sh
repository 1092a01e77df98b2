#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02x
timeout 300 python tools/copy_floor.py 64 8 2>&1 | tee gpurun_out/r02x/floor.txt
timeout 300 python tools/group_cost.py 32 32 2>&1 | tee gpurun_out/r02x/gc.txt
timeout 300 python tools/group_cost.py 64 8 2>&1 | tee -a gpurun_out/r02x/gc.txt
timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q 2>&1 | tail -3 | tee gpurun_out/r02x/pipe.txt
