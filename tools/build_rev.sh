#!/usr/bin/env bash
# Build libwlbcp.so of a git revision into var/lib<name>.so (A/B experiments):
#   tools/build_rev.sh <rev> <name>
set -eu
rev=$1; name=$2
root="$(cd "$(dirname "$0")/.." && pwd)"
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2503_17924_b200/csrc paper_2503_17924_b200/build.py include | tar -x -C "$tmp"
mkdir -p "$root/var"
WLB_LIB_OUT="$root/var/lib$name.so" python "$tmp/paper_2503_17924_b200/build.py" > /dev/null
rm -rf "$tmp"
echo "$root/var/lib$name.so"
