#!/bin/bash
cd "$(dirname "$0")/.."
for r in 1 2 3; do for v in old new; do
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 0 3000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so HB_SWEEP_NMAX=4 timeout 120 python tools/kernel_sweep.py 1000 | cut -c60-100 | sed "s/^/[$v N4K1] /"
done; done
