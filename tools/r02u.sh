#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/pcie2d_probe.py 2>&1 | tee gpurun_out/pcie2d.txt
timeout 120 python tools/pcie_probe.py 2>&1 | tee -a gpurun_out/pcie2d.txt
