#!/usr/bin/env bash
# Same-box A/B at N=1: bench (7B and GQA) and the single-32K-document probe for
# library builds var/lib<name>.so: tools/ab_n1.sh <out> A B ...
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/$1; shift
mkdir -p $out
for rep in 1 2; do
  for n in "$@"; do
    export WLB_LIB_PATH=var/lib$n.so
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --clock-ms 0 > $out/b7_${n}_$rep.json 2>&1
    timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --clock-ms 0 --shape llama70b-gqa > $out/bg_${n}_$rep.json 2>&1
    timeout 120 python tools/probe_attn.py --single --iters 8 > $out/p_${n}_$rep.txt 2>&1
  done
done
unset WLB_LIB_PATH
for n in "$@"; do for rep in 1 2; do
  python -c "
import json
a=json.loads(open('$out/b7_${n}_$rep.json').read().strip().splitlines()[-1])['value']
b=json.loads(open('$out/bg_${n}_$rep.json').read().strip().splitlines()[-1])['value']
print('$n $rep bench7b', a, 'gqa', b, 'probe', open('$out/p_${n}_$rep.txt').read().strip().replace(chr(10),' | '))
" 2>&1 | tail -1
done; done
