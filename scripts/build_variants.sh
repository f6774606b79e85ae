#!/bin/bash
# Build experimental variants of the library (compile-time knobs) into build/variants/.
# usage: scripts/build_variants.sh name:"-DFLAG=1 -DX=2" ...
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -shared -Xcompiler -fPIC $flags -o build/variants/lib_$name.so paper_1804_10062_b200/csrc/qmsort_gpu.cu \
    > build/variants/$name.log 2>&1 &
done
wait
ls -la build/variants/*.so
