for r in 1 2; do
  timeout 120 python tools/kernel_sweep.py 200 | sed "s/^/[tables] /" | cut -c1-170
  HB_RANKTOP_EXP=1 timeout 120 python tools/kernel_sweep.py 200 | sed "s/^/[ranktop] /" | cut -c1-170
done
HB_RANKTOP_EXP=1 HEOM_B200_LIB=$PWD/paper_1012_4382_b200/libheomb200_checked.so timeout 900 python -m pytest tests/test_gpu_fullstate.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
