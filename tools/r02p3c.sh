#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for rep in 1 2; do for n in p1 p1t; do WLB_LIB_PATH=var/lib$n.so timeout 300 python tools/short_profile.py > gpurun_out/sp_$n.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/sp_$n.jsonl'):
    try: d=json.loads(l)
    except: continue
    print('$n', d['mb'], d['strategy'], d['max_rank_ms'], d['tflops_per_gpu'])
"; done; done
WLB_LIB_PATH=var/libp1t.so timeout 600 python tools/config5.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print('p1t c5', d['iteration'], d['per_document_chosen'], [(x['strategy'][:7], x['tflops_per_gpu']) for x in d['sample']])
"
bash tools/ab_n1.sh p3c p1 p1t
