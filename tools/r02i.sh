#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/r02i; mkdir -p $out
WLB_LIB_PATH=var/libJ.so timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_scale.py tests/test_gpu_exchange.py -q -x > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
tail -2 $out/tests.txt
bash tools/ab_n1.sh ab6 I J
for n in I J; do
  WLB_LIB_PATH=var/lib$n.so timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/launches_gqa_$n.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --clock-ms 0 --shape llama70b-gqa > /dev/null 2>&1
done
