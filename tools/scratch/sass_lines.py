"""Join an ncu SASS source-page csv with nvdisasm line info: stall samples
and executed instructions per CUDA source line of one kernel."""
import csv, re, subprocess, sys, collections
cubin, func, csvp = sys.argv[1], sys.argv[2], sys.argv[3]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
start = dis.index(f".text.{func}:")
end = dis.find("//---------------------", start)
body = dis[start:end]
cur = None
amap = {}
for line in body.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m:
        amap[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvp)))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) >= len(hdr) and r[0].startswith("0x"):
        data.append(r)
base = int(data[0][0], 16)
agg = collections.defaultdict(lambda: [0.0, 0.0])
ts = ti = 0
for r in data:
    a = int(r[0], 16) - base
    k = amap.get(a, ("?", 0))
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    i = float(r[ix["Instructions Executed"]] or 0)
    agg[k][0] += s
    agg[k][1] += i
    ts += s
    ti += i
src = {}
for (f, l) in agg:
    pass
top = sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[4]) if len(sys.argv) > 4 else 40]
for (f, l), (s, i) in top:
    print(f"{100*s/ts:5.1f}% stall  {100*i/ti:5.1f}% inst  {f}:{l}")
