#!/usr/bin/env bash
cd "$(dirname "$0")/.."
WLB_LIB_PATH=var/libtrace.so timeout 120 python tools/bwd_trace.py --doc 256 --ndocs 128 --show 70 2>&1 | tee gpurun_out/bwd_trace_256.txt
