#!/usr/bin/env bash
# ncu --set full of the persistent 128-query backward on 16 x 2048-row documents (7B shape)
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/ncu_short; mkdir -p $out
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:attn_bwd3 -c 1 -o $out/bwd3_doc2048 python tools/probe_attn.py --doc 2048 --iters 1 > $out/ncu.log 2>&1
python tools/ncu_summary.py $out/bwd3_doc2048.ncu-rep > $out/bwd3_doc2048.summary.txt 2>&1
cat $out/bwd3_doc2048.summary.txt
