#!/bin/bash
# usage: tools/sweep.sh CONFIG "ENV1=a ENV2=b" "ENV1=c" ...   — one short bench per env combo
cfg=$1; shift
for combo in "$@"; do
  tag=$(echo "$combo" | tr ' =' '_-')
  env $combo timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sw_c${cfg}_$tag.log 2>&1
  python - "$cfg" "$combo" "gpurun_out/sw_c${cfg}_$tag.log" <<'PY'
import json, sys
cfg, combo, fn = sys.argv[1:4]
try:
    d = json.loads(open(fn).read().strip().splitlines()[-1])
    print(f"c{cfg} [{combo}] ms/step {d['ms_per_step']:.4f} val {d['value']:.3e} hbm {d['hbm_roofline_step']['frac']:.3f}",
          {k: round(x['ms_total'] / d['steps'], 3) for k, x in d['kernels'].items()})
except Exception as e:
    print(f"c{cfg} [{combo}] FAIL {e}", open(fn).read()[-500:])
PY
done
