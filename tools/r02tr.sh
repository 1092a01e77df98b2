#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for n in trace traceT traceN; do echo "== $n"; WLB_LIB_PATH=var/lib$n.so timeout 120 python tools/bwd_trace.py --doc 256 --ndocs 128 --show 40 2>&1; WLB_LIB_PATH=var/lib$n.so timeout 120 python tools/probe_attn.py --doc 256 --iters 8; done | tee gpurun_out/bwd_trace_256b.txt
