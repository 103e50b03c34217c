#!/bin/bash
# K1/K2 per-class ms per step of bench.py for the in-tree build and variant builds (QMC_LIB)
# usage: tools/variant_k1.sh CONFIG variant1 variant2 ...
c=$1; shift
mkdir -p gpurun_out/r2/var
QMC_ONE_STREAM=1 timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r2/var/c${c}_main.log 2>&1
for v in "$@"; do
  QMC_ONE_STREAM=1 QMC_LIB=$PWD/variants/libqmc_$v.so timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r2/var/c${c}_$v.log 2>&1
done
python tools/bench_summary.py gpurun_out/r2/var/c${c}_*.log
