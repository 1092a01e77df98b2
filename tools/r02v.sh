#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02v
timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q 2>&1 | tail -5 | tee gpurun_out/r02v/pipe.txt
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --clock-ms 0 > gpurun_out/r02v/b7.json 2>&1; tail -c 900 gpurun_out/r02v/b7.json
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --clock-ms 0 --shape llama70b-gqa > gpurun_out/r02v/bg.json 2>&1; tail -c 600 gpurun_out/r02v/bg.json
