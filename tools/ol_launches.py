"""Per-launch table (second half of the launches = the last repetition) of an
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv log of tools/one_layer.py.  usage: ol_launches.py <csv> [name filter]"""
import csv, sys
lines = open(sys.argv[1]).read().split('\n')
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[1:] if len(r) == len(hdr)]
ids = sorted(set(int(r[ix['ID']]) for r in data))
half = set(ids[len(ids) // 2:])
agg = {}
for r in data:
    if int(r[ix['ID']]) not in half: continue
    k = (int(r[ix['ID']]), r[ix['Kernel Name']][:50])
    agg.setdefault(k, {})[r[ix['Metric Name']]] = r[ix['Metric Value']]
flt = sys.argv[2] if len(sys.argv) > 2 else 'dsmpnn'
tot = 0
f = lambda m, k: float(m.get(k, '0').replace(',', ''))
for (i, n), m in sorted(agg.items()):
    t = f(m, 'gpu__time_duration.sum'); tot += t
    if flt in n:
        print(f"{i:4d} {n:50s} {t/1000:8.1f} us  rd {f(m,'dram__bytes_read.sum')/1e6:7.1f} MB"
              f" wr {f(m,'dram__bytes_write.sum')/1e6:7.1f} MB")
print("total us", tot / 1000)
