#!/bin/bash
# bench lines of the given configs (CS) under gpurun_out/$TAG
O=gpurun_out/${TAG:-r2s3/q}; mkdir -p $O
for c in ${CS:-5 3 2 4}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/c$c.log 2>&1
done
python tools/bench_summary.py $O/*.log
