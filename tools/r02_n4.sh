#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
bash tools/multi_run.sh r02
bash tools/ab_multi.sh
