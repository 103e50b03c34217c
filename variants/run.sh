#!/bin/bash
# usage: variants/run.sh v1 v2 ...   (each variants/libqmc_$v.so)
for v in "$@"; do
  cp variants/libqmc_$v.so paper_1501_06286_b200/libqmc.so
  echo "=== $v"
  timeout 900 python -m pytest tests -m gpu -x -q -k "small or config1 or worked or edge or deterministic or config2 or tables" > gpurun_out/pt_$v.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_$v.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1; echo "bench rc=$?"
  python - "$v" <<'PY'
import json,sys
v=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/bench_{v}.log").read().strip().splitlines()[-1])
    print(v, "ms/step %.3f"%d["ms_per_step"], "value %.3e"%d["value"], "hbm_frac %.3f"%d["hbm_roofline_step"]["frac"], {k:(round(x["ms_total"]/d["steps"],4)) for k,x in d["kernels"].items()}, "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"],3), d["clocks"])
except Exception as e:
    print("parse fail", e); print(open(f"gpurun_out/bench_{v}.log").read()[-2000:])
PY
done
