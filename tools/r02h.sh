#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/r02h; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -k "project or fused" > $out/tests.txt 2>&1; echo "rc=$?" >> $out/tests.txt
tail -30 $out/tests.txt
timeout 300 python tools/proj_bench.py > $out/proj_bench.jsonl 2>&1
cat $out/proj_bench.jsonl
# launch list of the fused path (no cuBLAS kernel may appear)
timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h/proj_launches.csv python -c "
import sys; sys.path.insert(0, '.')
import torch, paper_2503_17924_b200 as wl
from paper_2503_17924_b200.cp import project_qkv, shard_for_rank
plan = wl.build_shard_plan([[70000, 61072]], 8, 'per_document')
sh = shard_for_rank(plan, 0, 3)
x = torch.randn(131072, 4096, device='cuda', dtype=torch.bfloat16)
w = torch.randn(4096, 96 * 128, device='cuda', dtype=torch.bfloat16)
project_qkv(x, w, sh, 32, 32, 128, gather=True)
torch.cuda.synchronize()
" > gpurun_out/r02h/proj_ncu.log 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(l for l in open('gpurun_out/r02h/proj_launches.csv') if not l.startswith('==')))
names = [r[4] for r in rows[1:] if len(r) > 4]
print('launches:', names)
PY
