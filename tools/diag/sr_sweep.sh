#!/bin/bash
# config 5 (and 3) with K1's staged first rounds capped at SR rounds (QMC_K1_SR)
O=gpurun_out/${TAG:-r2s3/sr}; mkdir -p $O
for c in ${CS:-5}; do for sr in ${SRS:-0 2 4 7}; do
  QMC_K1_SR=$sr timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/c${c}_sr$sr.log 2>&1
done; done
python tools/bench_summary.py $O/*.log
