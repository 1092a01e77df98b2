#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for d in 256 512 1024; do for n in v4096 v1024 v512 v1; do WLB_LIB_PATH=var/lib$n.so timeout 120 python tools/probe_attn.py --doc $d --iters 8 | sed "s/^/$n doc$d /"; done; done
bash tools/ab_n1.sh v3thr2 v1024 v512 v1
