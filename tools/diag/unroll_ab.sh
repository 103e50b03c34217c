#!/bin/bash
# K1 scatter with batched group loads: main build (U = 4) vs variants (QMC_LIB) on configs 5, 3, 2
O=gpurun_out/${TAG:-r2s3/unroll}; mkdir -p $O
for c in ${CS:-5 3 2}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/c${c}_u4.log 2>&1
  for v in ${VS:-u6 u8}; do
    QMC_LIB=$PWD/variants/libqmc_$v.so timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/c${c}_$v.log 2>&1
  done
done
python tools/bench_summary.py $O/*.log
