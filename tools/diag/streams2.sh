mkdir -p gpurun_out/r2/streams2
for r in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/streams2/main_r$r.log 2>&1
  QMC_LIB=$PWD/variants/libqmc_two.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/streams2/two_r$r.log 2>&1
  QMC_ONE_STREAM=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/streams2/one_r$r.log 2>&1
done
python tools/bench_summary.py gpurun_out/r2/streams2/*.log
