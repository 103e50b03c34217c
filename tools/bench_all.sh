#!/bin/bash
# bench lines of the given configs (default: 2 5) into gpurun_out/$TAG/bench_c<c>.log
TAG=${TAG:-r2}
mkdir -p gpurun_out/$TAG
for c in ${@:-2 5}; do
  steps=20; [ $c -ge 3 ] && steps=5; [ $c -eq 4 ] && steps=20
  timeout 600 python bench.py --config $c --steps $steps --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_c$c.log 2>&1
  echo "c$c rc=$?"
done
python tools/bench_summary.py gpurun_out/$TAG/bench_c*.log
