#!/usr/bin/env bash
# Fresh calibration measurements on the final kernels; the SHIPPED tile
# models (fitted on the previous measurements) scored on them without
# re-fitting, and the re-fit from them.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/cal3; mkdir -p $out
timeout 1500 python tools/calibrate_tiles.py --hq 32 --hkv 32 --out $out/tiles_7b.json > $out/tiles_7b.log 2>&1
python tools/score_tiles.py $out/tiles_7b.json > $out/score_7b.json 2>&1
timeout 1800 python tools/calibrate_tiles.py --hq 64 --hkv 8 --out $out/tiles_gqa.json > $out/tiles_gqa.log 2>&1
python tools/score_tiles.py $out/tiles_gqa.json > $out/score_gqa.json 2>&1
cat $out/score_7b.json $out/score_gqa.json
