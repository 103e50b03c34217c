# K2 (and K1) time per pair vs batch size, one stream (does U stay in L2 for small batches?)
for B in 16 32 64 256; do
  QMC_ONE_STREAM=1 QMC_BATCH_PAIRS=$B timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bs_$B.log 2>&1
  python - $B <<'PY'
import json,sys
B=int(sys.argv[1]); d=json.loads(open(f"gpurun_out/bs_{B}.log").read().strip().splitlines()[-1])
print(B, "ms/step %.3f" % d["ms_per_step"], {k: round(1e3*x['ms_total']/d['steps']/512,4) for k,x in d['kernels'].items()}, "us/pair")
PY
done
