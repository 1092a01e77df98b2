#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
bash tools/ab_n1.sh ab8 K V2048 V8192 V16384
