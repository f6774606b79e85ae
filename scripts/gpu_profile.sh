#!/bin/bash
# Round profile capture: bench line, launch list, ncu --set full of one sort, other configs.
# usage: scripts/gpu_profile.sh <prefix>
cd "$(dirname "$0")/.."
pre=${1:-prof}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python bench.py > gpurun_out/${pre}_bench.json 2> gpurun_out/${pre}_bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${pre}_launches.csv python bench.py --quick --steps 2 --warmup 3 > gpurun_out/${pre}_ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:sample_kernel|count_kernel|colsum_kernel|plan_kernel|scatter_kernel|blocksort_tasks|init_level" -c 15 -o gpurun_out/${pre}_full python bench.py --quick --steps 1 --warmup 1 > gpurun_out/${pre}_ncu2.log 2>&1; echo ncu2=$?
for c in c3 c4a c4b c4c c4d c4e c5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/${pre}_cfg_$c.json 2>&1; echo $c=$?
done
