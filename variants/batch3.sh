v=$1; shift
cp variants/libqmc_$v.so paper_1501_06286_b200/libqmc.so
for cfg in "$@"; do
b=${cfg%:*}; ex=${cfg#*:}
env QMC_BATCH_PAIRS=$b $ex timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_${v}_$b.log 2>&1
python - $v $b "$ex" <<'PY'
import json,sys
v,b,ex=sys.argv[1:4]
d=json.loads(open(f"gpurun_out/b_{v}_{b}.log").read().strip().splitlines()[-1])
print(v,b,ex,"ms/step %.3f"%d["ms_per_step"], {k:(round(x["ms_total"]/d["steps"],4)) for k,x in d["kernels"].items()})
PY
done
