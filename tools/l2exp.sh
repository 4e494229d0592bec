for r in 1 2; do for x in 0 100000; do
  HB_EL_EXP=$x python tools/small_probe.py 0 3000 2>&1 | grep "end to end" | sed "s/^/[el<=$x] /"
  HB_EL_EXP=$x python tools/small_probe.py 1 1000 2>&1 | grep "end to end" | sed "s/^/[el<=$x] /"
done; done
HB_EL_EXP=100000 HB_SWEEP_NMAX=4 timeout 120 python tools/kernel_sweep.py 1000 | cut -c1-120 | sed "s/^/[el N4K1] /"
HB_EL_EXP=0 HB_SWEEP_NMAX=4 timeout 120 python tools/kernel_sweep.py 1000 | cut -c1-120 | sed "s/^/[mm4 N4K1] /"
HB_EL_EXP=100000 HB_SWEEP_NMAX=8 timeout 120 python tools/kernel_sweep.py 100 | cut -c1-120 | sed "s/^/[el N8K1] /"
HB_EL_EXP=100000 HEOM_B200_LIB=$PWD/paper_1012_4382_b200/libheomb200_checked.so timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
