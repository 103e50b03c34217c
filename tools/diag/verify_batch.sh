OUT=gpurun_out/v3; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -1 $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c5.log 2>&1
timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c2.log 2>&1
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c3.log 2>&1
timeout 300 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.log 2>&1
python tools/bench_summary.py $OUT/bench_*.log
