python tools/devinfo.py
for w in 0 1 2 8; do
  for i in 1 2; do HB_L2_WINDOW=$w timeout 120 python tools/kernel_sweep.py 200; done
done
HB_L2_WINDOW=1 HB_L2_HIT=0.6 timeout 120 python tools/kernel_sweep.py 200
HB_L2_WINDOW=2 HB_L2_HIT=0.5 timeout 120 python tools/kernel_sweep.py 200
