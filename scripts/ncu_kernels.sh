#!/bin/bash
# ncu --set full capture of the named kernels of one C2 sort (after a plain run exits 0).
# usage: scripts/ncu_kernels.sh <out-prefix> <kernel-regex> <count> [bench args]
cd "$(dirname "$0")/.."
pre=$1; rx=$2; cnt=$3; shift 3
mkdir -p gpurun_out
timeout 300 python bench.py --quick --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" > gpurun_out/${pre}_plain.json 2>&1 || { echo plain-failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -c $cnt -o gpurun_out/${pre} python bench.py --quick --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" > gpurun_out/${pre}_ncu.log 2>&1
echo ncu=$?
