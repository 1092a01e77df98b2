#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02t
for b in 0 1; do timeout 120 python tools/probe_attn.py --batch $b --iters 10; done 2>&1 | tee gpurun_out/r02t/probe.txt
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02t/seq0.csv python tools/probe_attn.py --batch 0 --iters 2 > gpurun_out/r02t/ncu.log 2>&1
echo rc=$?
