#!/bin/bash
# ncu --set full of the four stage kernels of one config-4 RK4 step under the
# given kernel knobs; leaves CSV pages (raw, source) in gpurun_out/<tag>_*.csv.
#   tools/ncu_one.sh <tag> <kernel-regex> ENV=.. ENV=..
tag=$1; kre=$2; shift 2
mkdir -p gpurun_out
env "$@" timeout 300 python tools/kernel_sweep.py 30 > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
env "$@" ncu --set full --clock-control none --import-source on -k regex:$kre -s 40 -c 4 \
    -o gpurun_out/$tag python tools/kernel_sweep.py 3 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu $tag rc=$?"
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_source.csv 2>/dev/null
rm -f gpurun_out/$tag.ncu-rep
