#!/bin/bash
# config-5 bench lines at several batch sizes (QMC_BATCH_PAIRS): the K1/K2
# persistent grids' tails per launch against the scratch size
OUT=${OUT:-gpurun_out/bs}; mkdir -p $OUT
for b in ${BS:-0 128 256 592 1024}; do
  if [ $b = 0 ]; then unset QMC_BATCH_PAIRS; else export QMC_BATCH_PAIRS=$b; fi
  timeout 400 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > $OUT/c5_b$b.log 2>&1
done
unset QMC_BATCH_PAIRS
python tools/bench_summary.py $OUT/*.log
