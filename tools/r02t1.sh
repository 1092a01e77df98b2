#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for n in t0 t1 t1p0 t0 t1 t1p0; do WLB_LIB_PATH=var/lib$n.so timeout 120 python tools/probe_attn.py --single --iters 8 | sed "s/^/$n /"; done
bash tools/ab_n1.sh tred2 t0 t1 t1p0
