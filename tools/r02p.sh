#!/usr/bin/env bash
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
for G in auto mb; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29741 tools/e2e_timeline_mp.py $G 2>&1 | grep -v "^\*\|OMP_NUM\|^$"
done | tee gpurun_out/e2e_timeline_n$N.txt
