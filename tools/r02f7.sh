#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/final9; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_tests.txt 2>&1; echo "all rc=$?" >> $out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "smoke rc=$?" >> $out/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench_n1.json 2> $out/bench_n1.err
timeout 600 python bench.py --steps 10 --warmup 3 --shape llama70b-gqa --no-cpu-baseline > $out/bench_n1_gqa.json 2> $out/bench_n1_gqa.err
timeout 900 python bench.py --steps 3 --warmup 3 --workload 128k --no-cpu-baseline > $out/bench_n1_128k.json 2> $out/bench_n1_128k.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/launches_llama7b.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --clock-ms 0 > $out/ncu_bench.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/launches_gqa.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --clock-ms 0 --shape llama70b-gqa > $out/ncu_bench_gqa.log 2>&1
timeout 900 python tools/config5.py > $out/config5.txt 2>&1
tail -n 2 $out/gpu_tests.txt; tail -n 1 $out/smoke.txt
for f in bench_n1 bench_n1_gqa bench_n1_128k bench_ref; do python -c "
import json
d=json.loads(open('$out/$f.json').read().strip().splitlines()[-1]); e=d.get('e2e') or {}; print('$f', d['value'], e.get('value'), e.get('ms_per_step'), (d.get('clocks') or {}).get('reasons'), (d.get('roofline') or {}).get('frac'))"; done
