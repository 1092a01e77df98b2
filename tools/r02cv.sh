#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/cv
WLB_LIB_PATH=var/libc1.so timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_scale.py tests/test_gpu_exchange.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -2
for n in c0 c1; do WLB_LIB_PATH=var/lib$n.so timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:dq_convert --clock-control none --csv python tools/probe_attn.py --single --iters 1 2>/dev/null | grep "gpu__time_duration\|dram__bytes" | sed "s/^/$n /" | cut -c1-220; done
bash tools/ab_n1.sh cv c0 c1
