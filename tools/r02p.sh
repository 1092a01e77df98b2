#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
i=0
for cfg in "WLB_XCHG_PUSH=dma WLB_CP_MEMOPS=1 WLB_CP_FUSED_SYNC=0" "WLB_XCHG_PUSH=covered WLB_CP_MEMOPS=1 WLB_CP_FUSED_SYNC=0" "WLB_XCHG_PUSH=dma WLB_CP_MEMOPS=0 WLB_CP_FUSED_SYNC=0" "WLB_XCHG_PUSH=dma WLB_CP_MEMOPS=1 WLB_CP_FUSED_SYNC=1"; do
  i=$((i+1))
  env $cfg timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2975$i tools/overlap_probe.py --seq 2 --groups 4 --reps 2 > gpurun_out/p$i.json 2> gpurun_out/p$i.err
  echo "$cfg rc=$? $(cut -c1-400 gpurun_out/p$i.json) $(grep -m1 'NativeError:' gpurun_out/p$i.err | cut -c1-200)"
done
