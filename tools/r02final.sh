#!/usr/bin/env bash
# Last-commit check on one B200: whole GPU suite, smoke, N=1 bench.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/final11; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_tests.txt 2>&1; echo "all rc=$?" >> $out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "smoke rc=$?" >> $out/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench_n1.json 2> $out/bench_n1.err
tail -n 2 $out/gpu_tests.txt; tail -n 1 $out/smoke.txt
python -c "
import json
d=json.loads(open('$out/bench_n1.json').read().strip().splitlines()[-1]); e=d.get('e2e') or {}; print('bench_n1', d['value'], e.get('value'), (d.get('clocks') or {}).get('reasons'), (d.get('roofline') or {}).get('frac'), d.get('gpu_launches'))"
