#!/bin/bash
# Compare one kernel family across library variants: ncu metrics per launch.
# usage: scripts/ncu_cmp.sh <kernel-regex> <count> [bench args]
cd "$(dirname "$0")/.."
rx=$1; cnt=$2; shift 2
M=gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,launch__grid_size
for lib in build/variants/lib_*.so; do
  name=$(basename $lib .so)
  QMSORT_GPU_LIB=$PWD/$lib timeout 600 ncu --metrics $M --clock-control none -k "regex:$rx" -c $cnt --csv python bench.py --quick --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncmp_$name.csv 2> gpurun_out/ncmp_$name.err
  echo "$name rc=$?"
done
