#!/usr/bin/env bash
# Round-2 N=1 measurement set: tile-model re-calibration (both shapes), bench
# lines (7B config 2, GQA shape), reference arm, ncu launch list + DRAM
# traffic of one bench step, one `ncu --set full` capture of the backward.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/m1; mkdir -p $out
timeout 1500 python tools/calibrate_tiles.py --hq 32 --hkv 32 --out $out/tiles_7b.json --model-out $out/b200_tiles_h32_kv32_d128.json > $out/tiles_7b.log 2>&1
timeout 1500 python tools/calibrate_tiles.py --hq 64 --hkv 8 --out $out/tiles_gqa.json --model-out $out/b200_tiles_h64_kv8_d128.json > $out/tiles_gqa.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench_n1.json 2> $out/bench_n1.err
timeout 900 python bench.py --steps 10 --warmup 3 --shape llama70b-gqa --no-cpu-baseline > $out/bench_n1_gqa.json 2> $out/bench_n1_gqa.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/launches_llama7b.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --clock-ms 0 > $out/ncu_bench.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/launches_gqa.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --clock-ms 0 --shape llama70b-gqa > $out/ncu_bench_gqa.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:attn_bwd3 -c 1 -o $out/bwd3_single32k python tools/probe_attn.py --single --iters 1 > $out/ncu_full.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:attn_fwd -c 1 -o $out/fwd_single32k python tools/probe_attn.py --single --iters 1 >> $out/ncu_full.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:qkv_proj -c 1 -o $out/proj_7b_cp8 python tools/proj_bench.py >> $out/ncu_full.log 2>&1
for f in bench_n1 bench_n1_gqa bench_ref; do tail -1 $out/$f.json | cut -c1-300; done
