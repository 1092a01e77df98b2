#!/usr/bin/env bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every
# device entry point on small cases; logs -> gpurun_out/sanitize/.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/sanitize
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 50 python tools/sanitize_case.py > "$out/$tool.log" 2>&1
  echo "$tool rc=$?" >> "$out/$tool.log"
  tail -4 "$out/$tool.log"
done
