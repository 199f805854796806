#!/bin/bash
# Same-box A/B of one CUDA source (dev tool, run under gpurun):
#   tools/ab.sh <repo-relative source> <alternative file> <command...>
# runs <command> on the current build, swaps the alternative in, rebuilds, runs it again.
set -u
src=$1; alt=$2; shift 2
echo "== A (current)"; "$@"
cp "$alt" "$src" && make -s -j 8 -C paper_1511_05174_b200/csrc > /dev/null 2>&1 || { echo "build failed"; exit 1; }
echo "== B ($alt)"; "$@"
