#!/bin/bash
cd "$(dirname "$0")/.."
for r in 1 2; do for v in old new4; do
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so timeout 120 python tools/kernel_sweep.py 200 | cut -c1-110 | sed "s/^/[$v config4] /"
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 1 1000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
done; done
cp exp_build/new4/libheomb200.so paper_1012_4382_b200/libheomb200.so
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > /tmp/t.log 2>&1; tail -1 /tmp/t.log; grep -A40 "^____" /tmp/t.log | head -50
