import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr is None or len(r)!=len(hdr): continue
    d=dict(zip(hdr,r))
    if d.get('Metric Name')!='gpu__time_duration.sum': continue
    v=float(d['Metric Value'].replace(',','')); u=d.get('Metric Unit','')
    v = v/1e3 if u in ('nsecond','ns') else (v*1e3 if u in ('msecond','ms') else v)
    n=d['Kernel Name']; n=n[:90]
    agg[n][0]+=1; agg[n][1]+=v
tot=sum(v[1] for v in agg.values())
for n,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:25]:
    print(f"{t:10.1f} us {100*t/tot:5.1f}% n={c:5d} {n}")
print("total us", tot)
