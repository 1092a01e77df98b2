#!/usr/bin/env bash
# Single-micro-batch CP exchange exposure vs SMs the persistent backward
# leaves to the exchange kernels (set_bwd_reserve_sms), 4 head groups.
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/rsv_n$N; mkdir -p $out
for s in 0 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 \
    tools/overlap_probe.py --seq $s --groups 4 --reserve 0 4 8 16 --reps 4 > $out/seq$s.json 2> $out/seq$s.err
  tail -1 $out/seq$s.json
done
