#!/bin/bash
# Memory-safety evidence without compute-sanitizer (closed on this pool):
#   1. the guard-zone tests (tests/test_guards_gpu.py) on the product build;
#   2. the whole GPU parity suite on the checked build (-DQMC_CHECK: bounds
#      checks of every computed row-slot, staged-slot, U and X index, trap on
#      violation), variants/libqmc_check.so loaded through QMC_LIB.
mkdir -p gpurun_out/r2
[ -f variants/libqmc_check.so ] || python -c "import sys; sys.path.insert(0,'paper_1501_06286_b200'); import build; build.build(out='variants/libqmc_check.so', extra=['-DQMC_CHECK'])"
timeout 900 python -m pytest tests/test_guards_gpu.py -m gpu -q > gpurun_out/r2/check_guards.log 2>&1
echo "guards rc=$?"; tail -1 gpurun_out/r2/check_guards.log
QMC_LIB=$PWD/variants/libqmc_check.so timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2/check_build.log 2>&1
echo "checked build rc=$?"; tail -1 gpurun_out/r2/check_build.log
grep -c "QMC_CHECK " gpurun_out/r2/check_build.log; grep "build flags" gpurun_out/r2/check_build.log | head -1; true
