mkdir -p gpurun_out/r2/grid
for g in 0 136 128 120 110; do
  QMC_K1_GRID=$g timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r2/grid/c5_g$g.log 2>&1
done
for g in 0 280 256 240; do
  QMC_K1_GRID=$g timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2/grid/c2_g$g.log 2>&1
done
python tools/bench_summary.py gpurun_out/r2/grid/*.log
