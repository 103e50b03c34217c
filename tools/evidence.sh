#!/bin/bash
# Round evidence on the GPU box (R=r01 by default): GPU tests, bench lines of
# every config, the launch list of the default bench command, one ncu --set
# full capture of K1 + K2 (config 2), per-launch DRAM traffic.  Summaries are
# copied into profiles/ by tools/evidence_collect.sh on the dev side.
R=${R:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${R}_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench_c2.jsonl 2> gpurun_out/${R}_bench_c2.err; echo "bench c2 rc=$?"
for c in 1 3 4 5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_bench_c$c.jsonl 2> gpurun_out/${R}_bench_c$c.err; echo "bench c$c rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/run_step.py --config 2 --steps 2 > gpurun_out/plainw.log 2>&1 && \
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_rows16|k_cols" -s 6 -c 2 \
  -o gpurun_out/${R}_full_c2 -f python tools/run_step.py --config 2 --steps 2 > gpurun_out/${R}_ncu_full.log 2>&1; echo "full rc=$?"
CFG=2 TAG=_${R} bash tools/prof_dram.sh
