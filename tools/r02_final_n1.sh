#!/usr/bin/env bash
# Final N=1 lines: config 2 (20 steps, full JSON), GQA shape, fixed-work 128K
# at N=1 (strong-scaling anchor), reference arm, smoke + GPU suite.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/final1; mkdir -p $out
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench_n1.json 2> $out/bench_n1.err
timeout 900 python bench.py --steps 10 --warmup 3 --shape llama70b-gqa --no-cpu-baseline > $out/bench_n1_gqa.json 2> $out/bench_n1_gqa.err
timeout 900 python bench.py --steps 3 --warmup 3 --workload 128k --no-cpu-baseline --no-e2e > $out/bench_n1_128k.json 2> $out/bench_n1_128k.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_tests.txt 2>&1; echo "rc=$?" >> $out/gpu_tests.txt
for f in bench_n1 bench_n1_gqa bench_n1_128k bench_ref; do tail -1 $out/$f.json | cut -c1-250; done; tail -n 2 $out/gpu_tests.txt; tail -n 1 $out/smoke.txt
