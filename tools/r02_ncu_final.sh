#!/usr/bin/env bash
# Round-2 ncu --set full refresh on the final kernels (persistent 128-query
# backward): one 32K document (7B shape), the forward on the same input, and
# one GQA 64q/8kv 32K document; summaries written next to the reports.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/ncu_final; mkdir -p $out
timeout 300 python tools/probe_attn.py --single --iters 3 > $out/probe.log 2>&1; echo "probe rc=$?" >> $out/probe.log
NCU="timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -c 1"
$NCU -k regex:attn_bwd3 -o $out/bwd3_single32k python tools/probe_attn.py --single --iters 1 > $out/ncu_full.log 2>&1
$NCU -k regex:attn_fwd -o $out/fwd_single32k python tools/probe_attn.py --single --iters 1 >> $out/ncu_full.log 2>&1
$NCU -k regex:attn_bwd3 -o $out/bwd3_gqa_single32k python tools/probe_attn.py --single --iters 1 --hq 64 --hkv 8 >> $out/ncu_full.log 2>&1
for r in bwd3_single32k fwd_single32k bwd3_gqa_single32k; do
  python tools/ncu_summary.py $out/$r.ncu-rep > $out/$r.summary.txt 2>&1
done
tail -3 $out/probe.log
grep -h -E "^==|tensor_cycles_active_realtime|dram__bytes|gpu__time" $out/*.summary.txt
