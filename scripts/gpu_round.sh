set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/h_launches.csv python bench.py --quick --steps 2 --warmup 1 > gpurun_out/h_ncu.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -c 30 -o gpurun_out/h_full python bench.py --quick --steps 1 --warmup 0 > gpurun_out/h_ncu2.log 2>&1; echo ncu2=$?
