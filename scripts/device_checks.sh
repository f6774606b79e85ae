#!/bin/bash
# The checked build (-DQMSORT_DEVICE_CHECKS=1: device-side bounds/invariant
# asserts that trap) over the small-size workload of every kernel path and the
# randomised stress suite.  compute-sanitizer is closed on the bench pool.
# usage: scripts/device_checks.sh   (needs build/variants/lib_checked.so:
#        scripts/build_variants.sh checked:"-DQMSORT_DEVICE_CHECKS=1")
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export QMSORT_GPU_LIB=$PWD/build/variants/lib_checked.so
timeout 1800 python scripts/sanitize_driver.py > gpurun_out/checks_driver.log 2>&1
echo "driver rc=$? $(tail -1 gpurun_out/checks_driver.log)"
QMSORT_STRESS_CASES=${QMSORT_STRESS_CASES:-400} timeout 1800 python -m pytest tests/test_gpu_stress.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_policy.py tests/test_gpu_boundary.py -q -x > gpurun_out/checks_pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/checks_pytest.log)"
