"""Stall samples per SASS region of one kernel in an ncu report (source page):
python tools/ncu_source.py REP REGEX [bucket]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 200
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Source" in r and "Address" in r)
data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
iS, iSrc, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
tot = sum(int(r[iS]) for r in data) or 1
print("samples", tot, "instr", sum(int(r[iE]) for r in data), "sass lines", len(data))
for k in range(0, len(data), B):
    seg = data[k:k + B]
    s = sum(int(r[iS]) for r in seg)
    e = sum(int(r[iE]) for r in seg)
    ops = {}
    for r in seg:
        t = r[iSrc].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] = ops.get(op, 0) + int(r[iE])
    top = sorted(ops.items(), key=lambda x: -x[1])[:6]
    print(f"{k:5d} samples {s:6d} ({100 * s / tot:4.1f}%) instr {e:9d}", top)
