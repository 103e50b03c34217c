#!/bin/bash
# A/B of K1's staged first rounds (QMC_K1_NOHYB=1: all rounds direct) on configs 5 and 3
O=gpurun_out/${TAG:-r2s3/hyb}; mkdir -p $O
for c in 5 3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/c${c}_hyb.log 2>&1
  QMC_K1_NOHYB=1 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/c${c}_nohyb.log 2>&1
done
python tools/bench_summary.py $O/*.log
