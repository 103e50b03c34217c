"""Per-stall-reason sample totals over a kernel's SASS, and the top N
instructions by samples with their dominant reasons:
python tools/ncu_stalls.py REP REGEX [N]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Source" in r and "Address" in r)
data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
reason_cols = [i for i, h in enumerate(hdr) if "(All Samples)" not in h and ("stall" in h.lower())]
iS, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
tot = {}
for r in data:
    for i in reason_cols:
        try:
            tot[hdr[i]] = tot.get(hdr[i], 0) + float(r[i] or 0)
        except ValueError:
            pass
T = sum(int(r[iS]) for r in data) or 1
print("total samples", T)
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:14]:
    print(f"  {k[:60]:60s} {v:10.0f} {100*v/T:5.1f}%")
top = sorted(range(len(data)), key=lambda i: -int(data[i][iS]))[:N]
for i in sorted(top):
    r = data[i]
    rs = sorted(((float(r[c] or 0), hdr[c]) for c in reason_cols if r[c] not in ("", "0")), reverse=True)[:3]
    print(f"{i:5d} {int(r[iS]):6d} {r[iSrc][:60]:60s}", [(h.replace('Warp Stall Sampling','').strip()[:28], int(v)) for v, h in rs])
