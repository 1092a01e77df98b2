set -u
mkdir -p gpurun_out/cal
timeout 600 python -m pytest tests/test_gpu_shard.py -q -x > gpurun_out/cal/shard_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/cal/shard_tests.txt
timeout 300 python tools/calibrate_tiles.py --quick --out gpurun_out/cal/quick.json > gpurun_out/cal/quick.log 2>&1 || { echo quick failed; tail -30 gpurun_out/cal/quick.log; exit 1; }
timeout 1500 python tools/calibrate_tiles.py --hq 32 --hkv 32 --out gpurun_out/cal/tiles_7b.json --model-out gpurun_out/cal/b200_tiles_h32_kv32_d128.json > gpurun_out/cal/tiles_7b.log 2>&1
timeout 1500 python tools/calibrate_tiles.py --hq 64 --hkv 8 --out gpurun_out/cal/tiles_gqa.json --model-out gpurun_out/cal/b200_tiles_h64_kv8_d128.json > gpurun_out/cal/tiles_gqa.log 2>&1
tail -5 gpurun_out/cal/shard_tests.txt; tail -60 gpurun_out/cal/tiles_7b.log
