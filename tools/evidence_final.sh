#!/bin/bash
# Final evidence of the round on the GPU box (product build in-tree, checked
# build in variants/): GPU suite, smoke, bench lines c1-c5 (c5 = the default
# with CPU baseline and e2e), reference arm, checked build + guards, the c5
# launch list of the bench command and one ncu --set full of K1/K2 (c5).
EV=${EV:-gpurun_out/fin2}; mkdir -p $EV
timeout 1200 python -m pytest tests -m gpu -q > $EV/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -1 $EV/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $EV/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $EV/bench_default.log 2>&1; echo "bench default rc=$?"
timeout 300 python bench.py --impl reference > $EV/ref_default.log 2>&1; echo "ref rc=$?"
timeout 200 python bench.py --config 1 --steps 50 --warmup 5 > $EV/bench_c1.log 2>&1
timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > $EV/bench_c2.log 2>&1
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > $EV/bench_c3.log 2>&1
timeout 300 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > $EV/bench_c4.log 2>&1
python tools/bench_summary.py $EV/bench_*.log > $EV/bench_summary.txt
bash tools/check_build.sh > $EV/check.txt 2>&1; cp gpurun_out/r2/check_*.log $EV/ 2>/dev/null
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $EV/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $EV/launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $EV/ncu_launch.log 2>&1
echo "launch list rc=$?"
CFG=5 T=256 S=3 C=2 K="k_rows16|k_cols" OUT=$EV/full_c5 bash tools/prof_k.sh
