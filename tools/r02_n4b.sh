#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/n4b_n$N; mkdir -p $out
for s in 0 2; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2971$s tools/overlap_probe.py --seq $s --groups 1 4 > $out/overlap_s$s.json 2> $out/overlap_s$s.err
cat $out/overlap_s$s.json
done
timeout 400 python bench.py --gpus $N --steps 5 --warmup 3 > $out/bench.json 2> $out/bench.err
timeout 400 python bench.py --gpus $N --steps 5 --warmup 3 --workload 128k --shape llama70b-gqa --no-e2e > $out/bench_gqa.json 2> $out/bench_gqa.err
tail -c 400 $out/bench.json; tail -c 300 $out/bench_gqa.json
