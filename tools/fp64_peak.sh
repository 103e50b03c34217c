#!/bin/bash
# measured fp64 peak with the SM clock sampled during the run -> gpurun_out/fp64_peak.json
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > gpurun_out/fp64_clocks.csv &
SMI=$!
sleep 1
/tmp/fp64_peak > gpurun_out/fp64_peak_raw.json
rc=$?
kill $SMI
python - <<'PY'
import json, statistics
d = json.load(open("gpurun_out/fp64_peak_raw.json"))
rows = [l.split(",") for l in open("gpurun_out/fp64_clocks.csv") if l.strip()]
sm = [float(r[0]) for r in rows]; pw = [float(r[2]) for r in rows]
load = [s for s, p in zip(sm, pw) if p > 300] or sm
d["clocks"] = {"sm_mhz_median_under_load": statistics.median(load), "samples": len(sm),
               "power_w_max": max(pw), "reasons_seen": sorted({r[3].strip() for r in rows})}
d["fp64_tflops_fma_at_max_clock_model"] = 2 * d["dfma_inst_per_s"] / 1e12 * d["sm_max_mhz"] / d["clocks"]["sm_mhz_median_under_load"]
json.dump(d, open("gpurun_out/fp64_peak.json", "w"), indent=1)
print(json.dumps(d))
PY
exit $rc
