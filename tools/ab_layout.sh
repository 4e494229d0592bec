# A/B: plane layout (scratch/plane) vs pair layout (this tree): timing + ncu of the 4 stage kernels
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  (cd scratch/plane && timeout 120 python tools/kernel_sweep.py 200 | sed 's/^/plane /')
  timeout 120 python tools/kernel_sweep.py 200 | sed 's/^/pair  /'
done
for v in plane pair; do
  d=.; [ $v = plane ] && d=scratch/plane
  (cd $d && timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_mm4 -s 8 -c 4 \
      -o /tmp/prof_$v python tools/kernel_sweep.py 3 > /tmp/ncu_$v.log 2>&1); echo "ncu $v rc=$?"
  ncu -i /tmp/prof_$v.ncu-rep --page raw --csv > $O/ab_${v}_raw.csv 2>/dev/null
done
