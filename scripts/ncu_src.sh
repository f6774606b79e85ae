#!/bin/bash
# ncu source-level capture (SASS + stall sampling) of one kernel per library variant.
# usage: scripts/ncu_src.sh <kernel-regex> [bench args]
cd "$(dirname "$0")/.."
rx=$1; shift
for lib in build/variants/lib_*.so; do
  name=$(basename $lib .so)
  QMSORT_GPU_LIB=$PWD/$lib timeout 600 ncu --section SourceCounters --section WarpStateStats --clock-control none -k "regex:$rx" -c 1 -o gpurun_out/nsrc_$name python bench.py --quick --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" > gpurun_out/nsrc_$name.log 2>&1
  echo "$name rc=$?"
done
