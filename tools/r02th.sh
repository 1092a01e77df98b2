#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for d in 128 256 384; do for t in 1000000 0; do timeout 120 python tools/probe_attn.py --doc $d --iters 8 --v3-min-rows $t | sed "s/^/thr$t doc$d /"; done; done
