mkdir -p gpurun_out/r2/bs5
for bp in 32 64 128 256; do
  QMC_BATCH_PAIRS=$bp timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/r2/bs5/c5_bp$bp.log 2>&1
done
python tools/bench_summary.py gpurun_out/r2/bs5/*.log
