#!/usr/bin/env bash
cd "$(dirname "$0")/.."
bash tools/cal_run.sh > /dev/null 2>&1
tail -3 gpurun_out/cal/shard_tests.txt
timeout 1500 bash tools/debug_checks.sh
