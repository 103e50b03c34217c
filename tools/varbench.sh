#!/bin/bash
# bench lines of the in-tree build and of variant builds (QMC_LIB) for the
# given configs: VARS="a b" CFGS="5 2" OUT=dir bash tools/varbench.sh
OUT=${OUT:-gpurun_out/var}; mkdir -p $OUT
for c in ${CFGS:-5 2}; do
  timeout 400 python bench.py --config $c --steps ${STEPS:-6} --warmup 3 --no-cpu-baseline > $OUT/c${c}_main.log 2>&1
  for v in $VARS; do
    QMC_LIB=$PWD/variants/libqmc_$v.so timeout 400 python bench.py --config $c --steps ${STEPS:-6} --warmup 3 --no-cpu-baseline > $OUT/c${c}_$v.log 2>&1
  done
done
python tools/bench_summary.py $OUT/*.log
