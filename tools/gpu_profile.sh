#!/bin/bash
# One GPU round trip: gpu tests, launch list, one ncu --set full capture of the
# four stage kernels (summarised into profiles/r1_stage_kernels.json on the box,
# which the bench reads for roofline.traffic), then the bench.  Everything the
# caller needs lands in gpurun_out/ (the .ncu-rep is reduced to CSV pages).
#   tools/gpu_profile.sh <kernel-regex> [bench args...]
set -u
K=${1:-k_mm4}; shift || true
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest=$?" | tee -a $O/pytest_gpu.log
python bench.py --steps 20 --warmup 20 --no-cpu-baseline --no-eta "$@" > /dev/null 2>&1; echo "plain=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -s 80 -c 40 --csv \
    --log-file $O/launches.csv python bench.py --steps 20 --warmup 20 --no-cpu-baseline --no-eta "$@" > $O/ncu1.log 2>&1
echo "ncu1=$?"
python bench.py --steps 3 --warmup 20 --no-cpu-baseline --no-eta "$@" > /dev/null 2>&1; echo "plain2=$?"
ncu --set full --clock-control none --import-source on -k regex:$K -s 80 -c 4 -o $O/prof \
    python bench.py --steps 3 --warmup 20 --no-cpu-baseline --no-eta "$@" > $O/ncu2.log 2>&1
echo "ncu2=$?"
ncu -i $O/prof.ncu-rep --page raw --csv > $O/prof_raw.csv 2>/dev/null
ncu -i $O/prof.ncu-rep --page details --csv > $O/prof_details.csv 2>/dev/null
ncu -i $O/prof.ncu-rep --page source --csv --print-source sass > $O/prof_source.csv 2>/dev/null
rm -f $O/prof.ncu-rep
python tools/ncu_summary.py $O/prof_raw.csv profiles/r1_stage_kernels.json --n-ado 319770 > /dev/null && \
    cp profiles/r1_stage_kernels.json $O/stage_kernels.json
python bench.py "$@" > $O/bench.json 2> $O/bench.err; echo "bench=$?"
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench_ref=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
tail -2 $O/pytest_gpu.log
