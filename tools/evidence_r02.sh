#!/bin/bash
# Round-2 evidence on the GPU box: checked build + guards, the c5 launch list
# of the bench command, one ncu --set full capture of K1/K2 at the bench's
# batch (c5, 64 pairs per launch), per-launch DRAM traffic.
EV=${EV:-gpurun_out/r2/ev2}; mkdir -p $EV
bash tools/check_build.sh
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $EV/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $EV/launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $EV/ncu_launch.log 2>&1
echo "launch list rc=$?"
CFG=5 T=256 S=3 C=2 K="k_rows16|k_cols" OUT=$EV/full_c5 bash tools/prof_k.sh
