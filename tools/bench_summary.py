"""One line per bench JSON log: ms/step, value, HBM fraction, dominant-kernel
roofline, e2e and per-class ms per step (reads gpurun_out/bench_*.log)."""
import glob
import json
import sys

for fn in sorted(sys.argv[1:] or glob.glob("gpurun_out/bench_*.log")):
    try:
        d = json.loads(open(fn).read().strip().splitlines()[-1])
        ks = {k: round(x["ms_total"] / d["steps"], 4) for k, x in d.get("kernels", {}).items()}
        print(fn, "ms/step %.4f" % d["ms_per_step"], "val %.3e" % d["value"],
              "hbm %.3f" % d["hbm_roofline_step"]["frac"],
              "roof %s %.3f" % (d["roofline"]["kernel"], d["roofline"]["frac"]),
              "e2e %.3e" % d["e2e"]["value"], ks, "clk", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
    except Exception as e:  # noqa: BLE001
        print(fn, "parse fail:", e, open(fn).read()[-800:])
