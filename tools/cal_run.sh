#!/usr/bin/env bash
# Tile-model calibration on one B200 (both head shapes) + the short-document profile.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/cal
timeout 600 python -m pytest tests/test_gpu_shard.py -q -x > gpurun_out/cal/shard_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/cal/shard_tests.txt
timeout 300 python tools/short_profile.py > gpurun_out/cal/short_profile.jsonl 2>&1
timeout 1500 python tools/calibrate_tiles.py --hq 32 --hkv 32 --out gpurun_out/cal/tiles_7b.json --model-out gpurun_out/cal/b200_tiles_h32_kv32_d128.json > gpurun_out/cal/tiles_7b.log 2>&1
timeout 1500 python tools/calibrate_tiles.py --hq 64 --hkv 8 --out gpurun_out/cal/tiles_gqa.json --model-out gpurun_out/cal/b200_tiles_h64_kv8_d128.json > gpurun_out/cal/tiles_gqa.log 2>&1
tail -3 gpurun_out/cal/shard_tests.txt; cat gpurun_out/cal/short_profile.jsonl | cut -c1-300; head -80 gpurun_out/cal/tiles_7b.log
