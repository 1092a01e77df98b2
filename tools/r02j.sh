#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/r02j; mkdir -p $out
timeout 300 python tools/split_probe.py > $out/split.jsonl 2>&1
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/short_launches.csv python tools/short_profile.py --ranks 1 --reps 1 > $out/short_ncu.log 2>&1
cat $out/split.jsonl
