#!/bin/bash
cd "$(dirname "$0")/.."
for r in 1 2; do for v in v0 a15_60 a20_62 a10_66; do
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so timeout 120 python tools/kernel_sweep.py 200 2>&1 | grep ms_per | cut -c1-150 | sed "s/^/[$v] /"
done; done
for v in v0 a15_60; do
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 1 1000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so HB_SWEEP_PREC=single timeout 120 python tools/kernel_sweep.py 200 2>&1 | grep ms_per | cut -c1-150 | sed "s/^/[$v single] /"
done
