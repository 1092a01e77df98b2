#!/usr/bin/env bash
# The checked build (-DWLB_DEBUG_CHECKS: device-side bounds / invariant traps)
# run through the whole -m gpu suite and smoke(); compute-sanitizer is closed
# on the GPU pool.  Build here: WLB_LIB_OUT=var/libdbg.so WLB_NVCC_EXTRA=-DWLB_DEBUG_CHECKS
#   python -m paper_2503_17924_b200.build ; run on the box: tools/debug_checks.sh
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/debug_checks; mkdir -p $out
export WLB_LIB_PATH=var/libdbg.so
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_tests.txt 2>&1; echo "rc=$?" >> $out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1; echo "rc=$?" >> $out/smoke.txt
tail -n 3 $out/gpu_tests.txt; tail -n 3 $out/smoke.txt
