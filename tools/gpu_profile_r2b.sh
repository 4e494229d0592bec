#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-eta --no-sweep --no-reference"
$B > /dev/null 2>&1; echo "plain=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches.csv $B > $O/ncu_launches.log 2>&1; echo "ncu-launches=$?"
HB_SWEEP_NMAX=6 HB_SWEEP_K=0 python tools/kernel_sweep.py 30 > /dev/null 2>&1; echo sweep=$?
HB_SWEEP_NMAX=6 HB_SWEEP_K=0 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_mm4ab -s 40 -c 4 -o /tmp/ab python tools/kernel_sweep.py 5 > $O/ncu_ab.log 2>&1; echo "ncu-ab=$?"
ncu -i /tmp/ab.ncu-rep --page raw --csv > $O/r2_ab_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/r2_ab_raw.csv $O/r2_k_mm4ab_k0twin.json --n-ado 1716 > /dev/null; echo sum=$?
python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1; echo smoke-launches=$?
