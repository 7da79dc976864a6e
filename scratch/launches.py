import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[hi+1:]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].replace('void ','')
    v = float(r[vi].replace(',',''))
    v *= {'nsecond':1e-3,'ns':1e-3,'usecond':1,'us':1,'msecond':1e3,'ms':1e3}.get(r[ui], 1)
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:60]:60s} n={cnt[k]:4d} total={v/1e3:9.3f} ms avg={v/cnt[k]:9.1f} us share={100*v/T:5.1f}%")
