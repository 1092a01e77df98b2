#!/usr/bin/env bash
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m 2>&1 | head -12
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29751 tools/pcie_multi.py 2>&1 | grep world | tee gpurun_out/pcie_multi_n$N.txt
