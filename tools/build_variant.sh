#!/bin/bash
# Build an experiment variant of libphoton.so with one source recompiled under
# extra nvcc flags:  tools/build_variant.sh <out.so> <source.cu> <flags...>
# (objects of the other sources come from paper_2411_02908_b200/_build)
set -e
OUT=$1; SRC=$2; shift 2
PKG=paper_2411_02908_b200
OBJ=/tmp/variant_$(basename $OUT .so).o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  -Iinclude -I$PKG/csrc --expt-relaxed-constexpr -diag-suppress 177 "$@" -c $PKG/csrc/$SRC -o $OBJ
OBJS=$(ls $PKG/_build/*.o | grep -v "/$SRC.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $OBJS $OBJ -lcudart -lcuda -ldl \
  -L/usr/local/cuda/lib64 -L/usr/local/cuda/lib64/stubs -Xlinker -rpath=/usr/local/cuda/lib64
echo $OUT
