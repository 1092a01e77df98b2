#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/fe
WLB_LIB_PATH=var/libf1.so timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_scale.py tests/test_gpu_exchange.py -x -q 2>&1 | tail -2
for rep in 1 2; do for n in f0 f1; do
for d in 256 1024 4096; do WLB_LIB_PATH=var/lib$n.so timeout 120 python tools/probe_attn.py --doc $d --iters 8 | sed "s/^/$n doc$d /"; done
WLB_LIB_PATH=var/lib$n.so timeout 300 python tools/short_profile.py > gpurun_out/fe/sp_$n.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/fe/sp_$n.jsonl'):
    try: d=json.loads(l)
    except: continue
    print('$n', d['mb'], d['strategy'], d['max_rank_ms'], d['tflops_per_gpu'], [r['fwd_ms'] for r in d['ranks']][:4])
"
done; done
bash tools/ab_n1.sh fe f0 f1
