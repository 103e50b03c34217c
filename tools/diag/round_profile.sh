# Round evidence for config 2 (bench workload): bench line, launch list of the
# bench command itself, one ncu --set full capture of K1 and K2 (warm).
R=${R:-r01}
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench_c2.jsonl 2> gpurun_out/${R}_bench_c2.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_ncu_launch.log 2>&1
echo launches rc=$?
timeout 300 python tools/run_step.py --config 2 --steps 2 > gpurun_out/plainw.log 2>&1 && \
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_rows16|k_cols" -s 6 -c 2 -o gpurun_out/${R}_full_c2 -f python tools/run_step.py --config 2 --steps 2 > gpurun_out/${R}_ncu_full.log 2>&1
echo full rc=$?
