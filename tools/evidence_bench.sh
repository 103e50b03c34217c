#!/bin/bash
# The driver's bench commands (default = config 5) plus the other configs' lines -> gpurun_out/$TAG
TAG=${TAG:-r2/final2}
mkdir -p gpurun_out/$TAG
timeout 900 python bench.py --impl reference > gpurun_out/$TAG/ref_default.log 2> gpurun_out/$TAG/ref_default.err; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/$TAG/bench_default.log 2> gpurun_out/$TAG/bench_default.err; echo "bench rc=$?"
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_c$c.log 2>&1; echo "c$c rc=$?"
done
python tools/bench_summary.py gpurun_out/$TAG/bench_*.log
