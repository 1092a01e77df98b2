#!/usr/bin/env bash
# which piece of the copy-engine / stream-memop exchange fails across GPUs
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/r02m_n$N; mkdir -p $out
run() {
  env "$@" timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=$((29800 + RANDOM % 100)) tests/cp_worker.py > $out/$1.log 2>&1
  echo "$* rc=$? $(grep -c 'CP OK' $out/$1.log) ok; $(grep -m2 -iE 'error|FAIL' $out/$1.log | cut -c1-300)"
}
run WLB_XCHG_PUSH=dma WLB_CP_MEMOPS=0 WLB_CP_FUSED_SYNC=0
run WLB_XCHG_PUSH=covered WLB_CP_MEMOPS=1 WLB_CP_FUSED_SYNC=0
run WLB_XCHG_PUSH=dma WLB_CP_MEMOPS=1 WLB_CP_FUSED_SYNC=0
run WLB_XCHG_PUSH=dma WLB_CP_MEMOPS=1 WLB_CP_FUSED_SYNC=1
