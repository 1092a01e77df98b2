#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for d in 128 256 384; do for t in 1000000 0; do WLB_LIB_PATH=var/libp1.so timeout 120 python tools/probe_attn.py --doc $d --iters 8 --v3-min-rows $t | sed "s/^/p1 thr$t doc$d /"; done; done
for d in 256 512; do for t in 1000000 0; do WLB_LIB_PATH=var/libp1.so timeout 120 python tools/probe_attn.py --hq 64 --hkv 8 --doc $d --iters 8 --v3-min-rows $t | sed "s/^/p1 gqa thr$t doc$d /"; done; done
for n in pold p1; do WLB_LIB_PATH=var/lib$n.so timeout 300 python tools/short_profile.py > gpurun_out/sp_$n.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/sp_$n.jsonl'):
    try: d=json.loads(l)
    except: continue
    print('$n', d['mb'], d['strategy'], d['max_rank_ms'], d['tflops_per_gpu'])
"; done
bash tools/ab_n1.sh p3 pold p1
