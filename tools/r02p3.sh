#!/usr/bin/env bash
cd "$(dirname "$0")/.."
# first a tiny guarded smoke of the persistent kernel
WLB_LIB_PATH=var/libp1.so timeout 120 python tools/probe_attn.py --doc 1024 --T 8192 --iters 2 2>&1 | tail -1
WLB_LIB_PATH=var/libp1.so timeout 600 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
WLB_LIB_PATH=var/libp1.so timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_exchange.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -2
for n in pold p0 p1; do for d in 512 1024 2048 32768; do WLB_LIB_PATH=var/lib$n.so timeout 120 python tools/probe_attn.py --doc $d --iters 8 | sed "s/^/$n doc$d /"; done; done
