"""Aggregate `ncu --page source --csv --print-source cuda,sass` output per CUDA source line:
instructions executed and stall samples.  usage: srcagg2.py file.csv [top]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None; hdr = None
agg = collections.defaultdict(lambda: [0, 0, ''])
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r[0] == 'Function Name': continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None or not r[0].isdigit(): continue
    ie = hdr.index('Instructions Executed'); ss = hdr.index('Warp Stall Sampling (All Samples)')
    k = (cur, int(r[0]))
    agg[k][2] = r[1].strip()[:90]
    try:
        agg[k][0] += int(r[ie] or 0); agg[k][1] += int(r[ss] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
print('total warp instr', tot, 'stall samples', ts)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]:15s}{k[1]:5d} {100*v[0]/max(tot,1):5.1f}% in {100*v[1]/max(ts,1):5.1f}% st | {v[2]}")
