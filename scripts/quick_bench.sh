#!/bin/bash
# Device-only C2 bench line + the phase ledger (one gpurun call while iterating on a kernel).
# usage: scripts/quick_bench.sh <tag> [bench args]
cd "$(dirname "$0")/.."
tag=$1; shift
mkdir -p gpurun_out
python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"; tail -c 400 gpurun_out/${tag}_bench.err
python - gpurun_out/${tag}_bench.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print(f"{d['value']:.2f} Gkeys/s {d['ms_per_step']:.3f} ms  " + " ".join(f"{k}={v['us']:.0f}({v['launches']})" for k,v in d['sort_roofline']['phases'].items()))
PY
