#!/bin/bash
cd "$(dirname "$0")/.."
for r in 1 2; do for v in v0 new; do
  HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 0 3000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
  HB_PROBE_NMAX=4 HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 1 2000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
  HB_PROBE_NMAX=5 HEOM_B200_LIB=$PWD/exp_build/$v/libheomb200.so python tools/small_probe.py 1 2000 2>&1 | grep "end to end" | sed "s/^/[$v] /"
done; done
for i in 1 2; do
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > /tmp/t.log 2>&1; tail -1 /tmp/t.log; grep -A40 "^____" /tmp/t.log | head -50
HEOM_B200_LIB=$PWD/paper_1012_4382_b200/libheomb200_checked.so timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > /tmp/t.log 2>&1; tail -1 /tmp/t.log; grep -A40 "^____" /tmp/t.log | head -50
done
