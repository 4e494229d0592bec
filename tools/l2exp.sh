#!/bin/bash
cd "$(dirname "$0")/.."
for r in 1 2; do for v in v0 pf1; do
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 0 3000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 1 1000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so HB_SWEEP_NMAX=4 timeout 120 python tools/kernel_sweep.py 1000 | cut -c1-120 | sed "s/^/[$v N4K1] /"
done; done
for v in v0 pf1big; do
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so timeout 120 python tools/kernel_sweep.py 200 2>&1 | grep ms_per | cut -c1-150 | sed "s/^/[$v] /"
done
