#!/bin/bash
# Build a variant of libheomb200.so with extra nvcc defines for the stage-kernel
# sources (hb_mm4.cu, plus any experimental csrc/hb_ep.cu):
#   tools/variant.sh NAME -DFOO=1 ...   ->  exp_build/NAME/libheomb200.so
# (load it with HEOM_B200_LIB=$PWD/exp_build/NAME/libheomb200.so).  Experiment tool.
set -e
cd "$(dirname "$0")/../paper_1012_4382_b200"
name=$1; shift
make -s libheomb200.so
mkdir -p ../exp_build/$name
F="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a -I../include"
extra=""
for src in hb_mm4 hb_ep hb_api; do
  [ -f csrc/$src.cu ] || continue
  nvcc $F "$@" -c csrc/$src.cu -o ../exp_build/$name/$src.o
  extra="$extra ../exp_build/$name/$src.o"
done
objs=$(ls build/*.o | grep -v -e hb_mm4.o -e hb_ep.o -e hb_api.o)
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../exp_build/$name/libheomb200.so $objs $extra -ldl
