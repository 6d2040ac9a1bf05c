"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes)."""
import csv, collections, sys

def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
    hdr = rows[hi]
    ix = {k: i for i, k in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        key = int(r[ix['ID']])
        d = per.setdefault(key, {'name': r[ix['Kernel Name']]})
        v = float(r[ix['Metric Value']].replace(',', ''))
        u = r[ix['Metric Unit']]
        scale = {'ns': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3, 'nsecond': 1e-3,
                 'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9, 'B': 1}.get(u, 1)
        d[r[ix['Metric Name']]] = v * scale
    return list(per.values())

if __name__ == '__main__':
    L = load(sys.argv[1])
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    L = L[skip:]
    tot = sum(d.get('gpu__time_duration.sum', 0) for d in L)
    for d in L:
        t = d.get('gpu__time_duration.sum', 0)
        rb = d.get('dram__bytes_read.sum', 0); wb = d.get('dram__bytes_write.sum', 0)
        print(f"{d['name'][:60]:60s} {t:10.1f} us  rd {rb/1e6:9.1f} MB  wr {wb/1e6:9.1f} MB  {((rb+wb)/t/1e3 if t else 0):7.0f} GB/s")
    print('total us', round(tot, 1), 'launches', len(L))
