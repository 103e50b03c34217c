for T in 128 256 1024; do
  QMC_ONE_STREAM=1 QMC_BATCH_PAIRS=64 timeout 300 python bench.py --config 2 --t $T --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ts_$T.log 2>&1
  python - $T <<'PY'
import json,sys
T=int(sys.argv[1]); d=json.loads(open(f"gpurun_out/ts_{T}.log").read().strip().splitlines()[-1])
pairs=T//2
print(T, {k: round(1e3*x['ms_total']/d['steps']/pairs,4) for k,x in d['kernels'].items()}, "us/pair")
PY
done
