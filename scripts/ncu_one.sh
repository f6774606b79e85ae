#!/bin/bash
# One `ncu --set full` capture of the first launch matching a kernel regex in a C2 sort;
# the report comes back in gpurun_out/<tag>.ncu-rep (read here with `ncu -i`).
# usage: scripts/ncu_one.sh <tag> <kernel-regex> [launch-skip] [bench args]
cd "$(dirname "$0")/.."
tag=$1; rx=$2; skip=${3:-0}; shift; shift; shift
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $skip -c 1 -f -o gpurun_out/$tag \
  python bench.py --quick --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" > gpurun_out/$tag.log 2>&1
echo "ncu rc=$?"
