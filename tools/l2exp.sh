#!/bin/bash
cd "$(dirname "$0")/.."
python tools/small_probe.py 0 3000 2>&1 | grep "end to end"
python tools/small_probe.py 1 1000 2>&1 | grep "end to end"
HB_SWEEP_NMAX=4 timeout 120 python tools/kernel_sweep.py 1000 | cut -c1-120
HB_SWEEP_NMAX=5 timeout 120 python tools/kernel_sweep.py 1000 | cut -c1-120
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
HEOM_B200_LIB=$PWD/paper_1012_4382_b200/libheomb200_checked.so timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
