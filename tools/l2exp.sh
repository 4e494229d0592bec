for k in stages auto stages auto; do python tools/small_probe.py 0 3000 0 $k 2>&1 | grep "end to end"; done
python tools/small_probe.py 1 500 0 auto 2>&1 | grep "end to end"
HEOM_B200_LIB=$PWD/paper_1012_4382_b200/libheomb200_checked.so timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
