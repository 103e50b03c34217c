# ncu --set full with warm caches (--cache-control none) on K1 and K2 of config ${CFG:-2}, mid-run
timeout 300 python tools/run_step.py --config ${CFG:-2} --steps 2 > gpurun_out/plainw.log 2>&1 && \
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"${KRE:-k_rows16|k_cols_x}" -s ${SKIP:-6} -c ${CNT:-2} -o gpurun_out/profw_c${CFG:-2} -f python tools/run_step.py --config ${CFG:-2} --steps 2 > gpurun_out/ncuw.log 2>&1
echo ncuw rc=$?
