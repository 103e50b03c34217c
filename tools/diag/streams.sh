mkdir -p gpurun_out/r2/streams
for r in 1 2; do for s in 0 1; do
  QMC_ONE_STREAM=$s timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/streams/c5_s${s}_r$r.log 2>&1
done; done
for s in 0 1; do QMC_ONE_STREAM=$s timeout 600 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2/streams/c4_s${s}.log 2>&1; done
python tools/bench_summary.py gpurun_out/r2/streams/*.log
