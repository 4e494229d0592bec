for m in 0 5 10 15 1 8 9 6; do
  HB_REV_EXP=$m timeout 120 python tools/kernel_sweep.py 200 | sed "s/^/[rev $m] /"
done
