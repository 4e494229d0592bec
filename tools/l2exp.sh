#!/bin/bash
cd "$(dirname "$0")/.."
for v in v0 ep; do HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so timeout 600 python tools/bitwise_dump.py /tmp/bw_$v.npz 2>&1 | tail -2; done
python tools/bitwise_dump.py --compare /tmp/bw_v0.npz /tmp/bw_ep.npz
for r in 1 2; do for v in v0 ep; do
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 0 3000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
done; done
for v in v0 ep; do
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 1 1000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so HB_SWEEP_NMAX=4 timeout 120 python tools/kernel_sweep.py 1000 | cut -c1-120 | sed "s/^/[$v N4K1] /"
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so timeout 120 python tools/kernel_sweep.py 100 2>&1 | grep ms_per | cut -c1-150 | sed "s/^/[$v] /"
done
