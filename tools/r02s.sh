#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29761 tools/nvlink_probe.py 2>&1 | grep -E "world|Error" | tee gpurun_out/nvlink_n$N.json
