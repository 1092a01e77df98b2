#!/usr/bin/env bash
# Unit-boundary timeline of the persistent 128-query backward (trace build).
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/trace; mkdir -p $out; rm -f $out/units*.txt
WLB_LIB_PATH=var/libT.so timeout 300 python tools/bwd3_trace.py --doc 2048 --ndocs 16 --units > $out/units.txt 2>&1
head -18 $out/units.txt
