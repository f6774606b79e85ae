#!/bin/bash
# Round profile capture: bench line, launch list, ncu --set full of one sort,
# the other configs, the mergesort path (bulk-copy merge passes) and the
# sharded path at P = 1 (folded exchange); profiles/summarize.py turns it into
# profiles/.
# usage: scripts/gpu_profile.sh <prefix>
cd "$(dirname "$0")/.."
pre=${1:-prof}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python bench.py > gpurun_out/${pre}_bench.json 2> gpurun_out/${pre}_bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${pre}_launches.csv python bench.py --quick --steps 2 --warmup 3 > gpurun_out/${pre}_ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:sample_kernel|count_kernel|colsum_kernel|plan_kernel|scatter_kernel|blocksort_tasks|tablesort_tasks|init_level" -c 15 -o gpurun_out/${pre}_full python bench.py --quick --steps 1 --warmup 1 > gpurun_out/${pre}_ncu2.log 2>&1; echo ncu2=$?
for c in c3 c4a c4b c4c c4d c4e c5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/${pre}_cfg_$c.json 2>&1; echo $c=$?
done
for c in c2 c3 c5; do
  timeout 300 python bench.py --algorithm mergesort --config $c --steps 3 --warmup 3 > gpurun_out/${pre}_merge_$c.json 2>&1; echo merge_$c=$?
  timeout 300 python bench.py --sharded --config $c --steps 8 --warmup 3 > gpurun_out/${pre}_sharded_$c.json 2>&1; echo sharded_$c=$?
done
timeout 600 ncu --set full --clock-control none -k "regex:merge_pass_bulk|merge_split" -c 4 -o gpurun_out/${pre}_merge_c3 python bench.py --quick --algorithm mergesort --config c3 --steps 1 --warmup 1 > gpurun_out/${pre}_ncu3.log 2>&1; echo ncu3=$?
timeout 600 ncu --set full --clock-control none -k "regex:merge_pass_kernel" -c 2 -o gpurun_out/${pre}_merge_c2 python bench.py --quick --algorithm mergesort --steps 1 --warmup 1 > gpurun_out/${pre}_ncu4.log 2>&1; echo ncu4=$?
# reports -> CSV on the box (gpurun copies back at most 64 MiB)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum
ncu -i gpurun_out/${pre}_full.ncu-rep --page raw --csv --metrics $M > gpurun_out/${pre}_full_raw.csv
for r in merge_c3 merge_c2; do
  ncu -i gpurun_out/${pre}_$r.ncu-rep --page raw --csv --metrics $M > gpurun_out/${pre}_${r}_raw.csv
  ncu -i gpurun_out/${pre}_$r.ncu-rep --page details --csv > gpurun_out/${pre}_${r}_details.csv
done
rm -f gpurun_out/${pre}_*.ncu-rep
du -sh gpurun_out
