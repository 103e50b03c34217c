#!/bin/bash
# config 5 with K2 on a green-context partition of G SMs (QMC_GREEN=G) vs one stream
O=gpurun_out/${TAG:-r2s3/green}; mkdir -p $O
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/c5_g0.log 2>&1
for G in ${GS:-16 24 32 40}; do
  QMC_GREEN=$G timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/c5_g$G.log 2>&1
done
python tools/bench_summary.py $O/*.log
