#!/bin/bash
# bench.py --sharded (device leg) against each library variant in build/variants/.
# usage: scripts/variants_sharded.sh [bench args...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in build/variants/lib_*.so; do
  name=$(basename $lib .so)
  QMSORT_GPU_LIB=$PWD/$lib timeout 300 python bench.py --sharded --steps 5 --warmup 3 "$@" > gpurun_out/vsh_$name.json 2> gpurun_out/vsh_$name.err
  echo "$name rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/vsh_$name.json').read().strip().splitlines()[-1]); print(round(d['value'],2), 'Gkeys/s', round(d['ms_per_step'],3), 'ms ledger', round(d['roofline']['ledger_bytes_over_nw'],2))" 2>&1 | tail -1)"
done
