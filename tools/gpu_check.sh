#!/usr/bin/env bash
# One GPU round trip: new parity tests, the whole -m gpu suite, smoke, bench N=1.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/${1:-check}
mkdir -p "$out"
export WLB_PARITY_LOG=$out/parity_scale.jsonl
rm -f "$WLB_PARITY_LOG"
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_scale.py -q -x > "$out/new_tests.txt" 2>&1; echo "new rc=$?" >> "$out/new_tests.txt"
timeout 1200 python -m pytest tests -m gpu -q > "$out/gpu_tests.txt" 2>&1; echo "all rc=$?" >> "$out/gpu_tests.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.txt" 2>&1; echo "smoke rc=$?" >> "$out/smoke.txt"
timeout 600 python bench.py --steps 10 --warmup 3 > "$out/bench_n1.json" 2> "$out/bench_n1.err"
tail -3 "$out"/*.txt
cat "$out/bench_n1.json"
