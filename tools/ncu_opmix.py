"""Executed-instruction mix (by SASS opcode) and stall samples per opcode of
one kernel in an ncu report: python tools/ncu_opmix.py REP REGEX"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Source" in r and "Address" in r)
data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
iS, iSrc, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
ops, smp = {}, {}
for r in data:
    t = r[iSrc].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[op] = ops.get(op, 0) + int(r[iE])
    smp[op] = smp.get(op, 0) + int(r[iS])
tot, ts = sum(ops.values()), sum(smp.values())
print("instr", tot, "samples", ts)
for op, n in sorted(ops.items(), key=lambda x: -x[1])[:28]:
    print(f"{op:10s} {n:12d} {100*n/tot:5.1f}%  stall-samples {100*smp[op]/ts:5.1f}%")
