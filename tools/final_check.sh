set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_tests.log 2>&1; echo tests=$?
HEOM_B200_LIB=$PWD/paper_1012_4382_b200/libheomb200_checked.so timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_tests_checked.log 2>&1; echo checked=$?
python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench=$?
python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo ref=$?
