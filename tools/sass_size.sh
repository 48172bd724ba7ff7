#!/bin/bash
# compile one csrc unit for sm_100a and print ptxas stats + SASS size per kernel
# usage: bash tools/sass_size.sh physics_f32 [extra nvcc flags]
R=$(cd $(dirname $0)/.. && pwd)
u=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I $R/include "$@" -Xptxas -v -c $R/paper_2502_08844_b200/csrc/$u.cu -o /tmp/$u.o 2>&1 | grep -E "error|registers|stack" | head -8
cuobjdump -sass /tmp/$u.o | grep -E "Function :|^\s+/\*[0-9a-f]+\*/" | awk '/Function :/{name=$NF; next} {c[name]++} END{for(n in c) print c[n], n}' | sort -rn | head -4
