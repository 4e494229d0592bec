#!/bin/bash
cd "$(dirname "$0")/.."
for r in 1 2; do for v in v0 ep epgs; do
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 0 3000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
done; done
HEOM_B200_LIB=$PWD/exp_build/epgs/libheomb200.so timeout 600 python tools/bitwise_dump.py /tmp/bw_g.npz 2>&1 | tail -1
HEOM_B200_LIB=$PWD/exp_build/v0/libheomb200.so timeout 600 python tools/bitwise_dump.py /tmp/bw_0.npz 2>&1 | tail -1
python tools/bitwise_dump.py --compare /tmp/bw_0.npz /tmp/bw_g.npz | grep -c identical
