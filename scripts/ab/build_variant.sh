#!/bin/bash
# Build libfastdog.so with another kernels.cu into $2 (same-box A/B: FDOG_LIB=$2 python bench.py ...)
set -e
KC=$1; OUTLIB=$2; T=$(mktemp -d)
cp -r paper_2111_10270_b200/csrc $T/csrc && cp $KC $T/csrc/kernels.cu
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Iinclude -I$T/csrc"
for s in plan.cpp solver.cpp; do nvcc $F -c -o $T/$s.o $T/csrc/$s & done
for s in kernels.cu compile_gpu.cu pack_gpu.cu; do nvcc $F -c -o $T/$s.o $T/csrc/$s & done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUTLIB $T/*.o -ldl
