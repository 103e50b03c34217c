mkdir -p gpurun_out
timeout 300 python tools/run_step.py --config 5 --t 192 --steps 2 > gpurun_out/p5plain.log 2>&1 && \
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_rows16|k_cols" -s 2 -c 2 -o gpurun_out/r01_full_c5 -f python tools/run_step.py --config 5 --t 192 --steps 2 > gpurun_out/p5ncu.log 2>&1
echo rc=$?
tail -3 gpurun_out/p5plain.log gpurun_out/p5ncu.log
