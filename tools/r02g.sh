#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
bash tools/ab_run.sh ab4 B G
bash tools/debug_checks.sh
