v=$1; shift
cp variants/libqmc_$v.so paper_1501_06286_b200/libqmc.so
for b in "$@"; do
QMC_BATCH_PAIRS=$b timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_${v}_$b.log 2>&1
python - $v $b <<'PY'
import json,sys
v,b=sys.argv[1:3]
d=json.loads(open(f"gpurun_out/b_{v}_{b}.log").read().strip().splitlines()[-1])
print(v,b,"ms/step %.3f"%d["ms_per_step"], {k:(round(x["ms_total"]/d["steps"],4)) for k,x in d["kernels"].items()})
PY
done
