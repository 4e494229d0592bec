#!/bin/bash
# One GPU round trip: gpu tests, bench, launch list, one ncu --set full capture of
# the stage kernels; summaries land in gpurun_out/ (the .ncu-rep is reduced to CSV
# pages on the box so the copy-back stays small).
#   tools/gpu_profile.sh <kernel-regex> [bench args...]
set -u
K=${1:-k_mm3}; shift || true
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest=$?" | tee -a $O/pytest_gpu.log
python bench.py "$@" > $O/bench.json 2> $O/bench.err; echo "bench=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -s 80 -c 40 --csv \
    --log-file $O/launches.csv python bench.py --steps 20 --warmup 20 --no-cpu-baseline "$@" > $O/ncu1.log 2>&1
echo "ncu1=$?"
ncu --set full --clock-control none --import-source on -k regex:$K -s 80 -c 4 -o $O/prof \
    python bench.py --steps 3 --warmup 20 --no-cpu-baseline "$@" > $O/ncu2.log 2>&1
echo "ncu2=$?"
ncu -i $O/prof.ncu-rep --page raw --csv > $O/prof_raw.csv 2>/dev/null
ncu -i $O/prof.ncu-rep --page details --csv > $O/prof_details.csv 2>/dev/null
ncu -i $O/prof.ncu-rep --page source --csv --print-source sass > $O/prof_source.csv 2>/dev/null
ls -la $O
rm -f $O/prof.ncu-rep
tail -2 $O/pytest_gpu.log
