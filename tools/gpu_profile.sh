#!/bin/bash
# One GPU round trip for the round's profile evidence (copied into profiles/ by
# the caller): the launch list of a short bench run, one ncu --set full capture
# of the four config-4 stage kernels with the default cache control (cold, the
# recipe's traffic figure) and one with --cache-control none (warm L2, what the
# steady state sees), reduced to CSV pages and JSON summaries.
#   tools/gpu_profile.sh <round-tag>
set -u
R=${1:-r2}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-eta --no-sweep --no-reference"
$B > /dev/null 2>&1; echo "plain=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches.csv $B \
    > $O/ncu_launches.log 2>&1; echo "ncu-launches=$?"
python tools/kernel_sweep.py 30 > /dev/null 2>&1; echo "sweep=$?"
for cc in all none; do
  ncu --set full --cache-control $cc --clock-control none --import-source on -k regex:k_mm4 -s 8 -c 4 \
      -o /tmp/prof_$cc python tools/kernel_sweep.py 3 > $O/ncu_full_$cc.log 2>&1; echo "ncu-full-$cc=$?"
  ncu -i /tmp/prof_$cc.ncu-rep --page raw --csv > $O/${R}_prof_${cc}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$cc.ncu-rep --page details --csv > $O/${R}_prof_${cc}_details.csv 2>/dev/null
  python tools/ncu_summary.py $O/${R}_prof_${cc}_raw.csv $O/${R}_stage_kernels_cache_$cc.json --n-ado 319770 > /dev/null
done
ncu -i /tmp/prof_all.ncu-rep --page source --csv --print-source sass > $O/${R}_prof_source.csv 2>/dev/null
echo done
