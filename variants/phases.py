import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
ix={h:i for i,h in enumerate(hdr)}
seen=set(); seq=[]
for r in data:
    a=r[ix["Address"]]
    if a in seen: continue
    seen.add(a); seq.append(r)
def f(r,k):
    try: return float(r[ix[k]])
    except: return 0.0
acc=0; start=seq[0][ix["Address"]][-5:]; tot=0; n=0; ops={}
for r in seq:
    s=r[ix["Source"]]
    acc+=f(r,"Warp Stall Sampling (All Samples)"); tot+=f(r,"Warp Stall Sampling (All Samples)"); n+=1
    op=s.split()[0] if s.split() else ''
    if op.startswith('@'): op=s.split()[1]
    op=op.split('.')[0]
    ops[op]=ops.get(op,0)+1
    if "BAR" in s or "EXIT" in s:
        top=sorted(ops.items(),key=lambda x:-x[1])[:6]
        print(start,"->",r[ix["Address"]][-5:], "samples",acc, "instrs", n, top)
        acc=0; n=0; start=r[ix["Address"]][-5:]; ops={}
print("total",tot)
