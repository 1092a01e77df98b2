#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
for s in 0 2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2974$s tools/push_probe.py $s 2>&1 | grep -E "world|Error" | cut -c1-600
done
