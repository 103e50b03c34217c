#!/bin/bash
# usage (on the GPU box): tools/gpu_check.sh [configs...]  — GPU tests + benches
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for c in "${@:-2}"; do
  extra=""; [ "$c" != 2 ] && extra="--no-cpu-baseline"
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 $extra > gpurun_out/bench_c$c.log 2>&1; echo "bench c$c rc=$?"
done
python tools/bench_summary.py
