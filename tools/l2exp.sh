#!/bin/bash
cd "$(dirname "$0")/.."
for r in 1 2; do for v in v0 s2x2; do
  HB_PROBE_NMAX=8 HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 0 2000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
  HB_PROBE_NMAX=7 HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 0 2000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
done; done
