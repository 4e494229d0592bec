#!/bin/bash
# Build a variant of libheomb200.so with extra nvcc defines for hb_mm4.cu only:
#   tools/variant.sh NAME -DFOO=1 ...   ->  exp_build/NAME/libheomb200.so
# (load it with HEOM_B200_LIB=$PWD/exp_build/NAME/libheomb200.so).  Experiment tool.
set -e
cd "$(dirname "$0")/../paper_1012_4382_b200"
name=$1; shift
make -s libheomb200.so
mkdir -p ../exp_build/$name
nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a -I../include "$@" \
  -c csrc/hb_mm4.cu -o ../exp_build/$name/hb_mm4.o
objs=$(ls build/*.o | grep -v hb_mm4.o)
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../exp_build/$name/libheomb200.so $objs ../exp_build/$name/hb_mm4.o -ldl
