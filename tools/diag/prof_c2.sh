# c2 profiling: one-stream bench (isolated per-kernel event times), launch list, ncu full of K1 + K2
QMC_ONE_STREAM=1 timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_onestream.log 2>&1
python tools/bench_summary.py gpurun_out/bench_c2_onestream.log
timeout 300 python tools/run_step.py --config ${CFG:-2} --steps 2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c${CFG:-2}.csv python tools/run_step.py --config ${CFG:-2} --steps 2 > gpurun_out/ncu1.log 2>&1
echo ncu1 rc=$?
python tools/launch_summary.py gpurun_out/launches_c${CFG:-2}.csv
timeout 300 python tools/run_step.py --config ${CFG:-2} --steps 1 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_rows16|k_cols_x}" -s ${SKIP:-2} -c ${CNT:-2} -o gpurun_out/prof_c${CFG:-2} -f python tools/run_step.py --config ${CFG:-2} --steps 1 > gpurun_out/ncu2.log 2>&1
echo ncu2 rc=$?
