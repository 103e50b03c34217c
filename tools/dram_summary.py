"""Per-launch DRAM bytes / L2 hit rate / time from a single-pass ncu csv."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r is not hdr and r[0] != "ID"]
per = OrderedDict()
for d in data:
    key = (d["ID"], d["Kernel Name"].split("(")[0][:40])
    per.setdefault(key, {})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
for (i, k), m in per.items():
    print(f"{i:>4} {k:40s}", "  ".join(f"{n.split('__')[1][:18]}={v} {u}" for n, (v, u) in m.items()))
