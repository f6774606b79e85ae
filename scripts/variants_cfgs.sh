#!/bin/bash
# Device-only bench lines of several configs against each library variant in build/variants/.
# usage: scripts/variants_cfgs.sh "<bench args of config 1>" "<bench args of config 2>" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in build/variants/lib_*.so; do
  name=$(basename $lib .so)
  for cfg in "$@"; do
    QMSORT_GPU_LIB=$PWD/$lib timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 $cfg 2>/dev/null | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read())
    print('$name', '$cfg', round(d['value'],2), 'Gkeys/s', round(d['ms_per_step'],3), 'ms', {k:round(v['us']) for k,v in d['sort_roofline']['phases'].items()})
except Exception as e: print('$name', '$cfg', 'parse fail', e)
"
  done
done
