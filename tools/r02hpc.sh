#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for rep in 1 2; do for n in h4 h2 h8; do
for d in 256 512; do WLB_LIB_PATH=var/lib$n.so timeout 120 python tools/probe_attn.py --doc $d --iters 8 | sed "s/^/$n doc$d /"; done
WLB_LIB_PATH=var/lib$n.so timeout 300 python tools/short_profile.py > gpurun_out/sp_$n.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/sp_$n.jsonl'):
    try: d=json.loads(l)
    except: continue
    print('$n', d['mb'], d['strategy'], d['max_rank_ms'], d['tflops_per_gpu'])
"
done; done
