import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
agg = collections.defaultdict(lambda: [0,0.0])
for r in rows[hdr_i+1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',','')); u = r[ui]
    v *= {'nsecond':1,'usecond':1e3,'msecond':1e6,'second':1e9}.get(u,1)
    name = r[ki].split('(')[0].split('<')[0]
    agg[name][0] += 1; agg[name][1] += v
tot = sum(a[1] for a in agg.values())
for k,(c,t) in sorted(agg.items(), key=lambda kv:-kv[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 12]:
    print(f"{k:45s} {c:7d} {t/1e6:10.2f} ms {100*t/tot:5.1f}%  avg {t/c/1e3:8.1f} us")
print('total kernel time', tot/1e6, 'ms; launches', sum(a[0] for a in agg.values()))
