#!/bin/bash
# Run bench.py (device leg only) against each library variant in build/variants/.
# usage: scripts/variants_bench.sh [bench args...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in build/variants/lib_*.so; do
  name=$(basename $lib .so)
  QMSORT_GPU_LIB=$PWD/$lib timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 "$@" > gpurun_out/var_$name.json 2> gpurun_out/var_$name.err
  echo "$name rc=$?"
  python - gpurun_out/var_$name.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ph=d['sort_roofline']['phases']
    print(f"  {d['value']:.2f} Gkeys/s {d['ms_per_step']:.3f} ms  " + " ".join(f"{k}={v['us']:.0f}" for k,v in ph.items()))
except Exception as e:
    print("  parse fail", e)
PY
done
