for f in 0 100000; do
  HB_FOLD_EXP=$f python tools/small_probe.py 0 3000 | sed "s/^/[fold<=$f] /"
  HB_FOLD_EXP=$f python tools/small_probe.py 1 2000 | sed "s/^/[fold<=$f] /"
  HB_FOLD_EXP=$f HB_SWEEP_NMAX=8 timeout 120 python tools/kernel_sweep.py 200 | sed "s/^/[fold<=$f] /" | cut -c1-150
done
