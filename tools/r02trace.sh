#!/usr/bin/env bash
# Unit-boundary cost of the persistent 128-query backward (trace build).
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/trace; mkdir -p $out
for doc in 512 1024 2048 4096 32768; do
  nd=$((32768 / doc))
  WLB_LIB_PATH=var/libT.so timeout 300 python tools/bwd3_trace.py --doc $doc --ndocs $nd --units >> $out/units.txt 2>&1
done
cat $out/units.txt
