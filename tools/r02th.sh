#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for d in 256 512 1024 2048 4096; do for t in 1000000 0; do timeout 120 python tools/probe_attn.py --hq 64 --hkv 8 --doc $d --iters 8 --v3-min-rows $t | sed "s/^/gqa thr$t doc$d /"; done; done
