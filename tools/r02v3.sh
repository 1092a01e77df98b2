#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for t in 320 0 320 0; do timeout 300 python tools/short_profile.py --v3-min-rows $t > gpurun_out/sp.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/sp.jsonl'):
    try: d=json.loads(l)
    except: continue
    print('thr$t', d['mb'], d['strategy'], d['max_rank_ms'], d['tflops_per_gpu'], [r['bwd_ms'] for r in d['ranks']][:4])
"; done
