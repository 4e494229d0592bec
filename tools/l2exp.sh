for r in 1 2; do
  timeout 120 python tools/kernel_sweep.py 200 | sed "s/^/[base] /" | cut -c1-170
  HB_ORDER_EXP=1 timeout 120 python tools/kernel_sweep.py 200 | sed "s/^/[A,top,t7] /" | cut -c1-170
done
