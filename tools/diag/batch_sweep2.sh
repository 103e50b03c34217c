OUT=gpurun_out/bs2; mkdir -p $OUT
for spec in "5 1024" "5 2048" "5 0" "3 0" "3 4096" "3 9824" "4 0" "4 512" "2 0" "2 512"; do
  set -- $spec
  if [ $2 = 0 ]; then unset QMC_BATCH_PAIRS; else export QMC_BATCH_PAIRS=$2; fi
  st=10; [ $1 = 2 ] && st=20; [ $1 = 4 ] && st=20
  timeout 400 python bench.py --config $1 --steps $st --warmup 3 --no-cpu-baseline > $OUT/c$1_b$2.log 2>&1
done
unset QMC_BATCH_PAIRS
python tools/bench_summary.py $OUT/*.log
