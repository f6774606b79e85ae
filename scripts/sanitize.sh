#!/bin/bash
# compute-sanitizer over the small-size workload of scripts/sanitize_driver.py
# (every dtype x comparator x kernel path); logs in gpurun_out/san_<tool>.log.
# usage: scripts/sanitize.sh [tool ...]   (default: memcheck racecheck synccheck)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tools=${@:-memcheck racecheck synccheck}
for t in $tools; do
  case $t in
    racecheck) sizes=1000,40000; extra="--racecheck-report all" ;;
    *) sizes=1000,40000,150007; extra="" ;;
  esac
  SAN_SIZES=$sizes timeout 2400 compute-sanitizer --tool $t $extra --target-processes all \
    --print-limit 200 python scripts/sanitize_driver.py > gpurun_out/san_$t.log 2>&1
  echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|failures' gpurun_out/san_$t.log | tr '\n' ' ')"
done
