import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
cur_file=None; hdr=None
agg=collections.defaultdict(lambda:[0,0,''])
for r in rows:
    if not r: continue
    if r[0]=='File Path': cur_file=r[1].split('/')[-1]; continue
    if r[0]=='Line No': hdr=r; continue
    if r[0]=='Function Name' or hdr is None: continue
    if r[0].isdigit() and len(r)>=2:
        line=(cur_file,int(r[0])); agg[line][2]=r[1].strip()[:80]
        try:
            agg[line][0]+=int(r[hdr.index('Instructions Executed')] or 0); agg[line][1]+=int(r[hdr.index('Warp Stall Sampling (All Samples)')] or 0)
        except Exception: pass
tot=sum(v[0] for v in agg.values()); ts=sum(v[1] for v in agg.values())
print('total instr', tot, 'samples', ts)
n=int(sys.argv[2]) if len(sys.argv)>2 else 40
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][0])[:n]:
    print(f"{k[0]:16s}{k[1]:5d} {100*v[0]/tot:5.1f}% instr {100*v[1]/max(ts,1):5.1f}% stall | {v[2]}")
print('--- by stall')
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][1])[:15]:
    print(f"{k[0]:16s}{k[1]:5d} {100*v[0]/tot:5.1f}% instr {100*v[1]/max(ts,1):5.1f}% stall | {v[2]}")
