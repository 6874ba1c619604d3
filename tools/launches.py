"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
gi = h.index('Grid Size') if 'Grid Size' in h else None
agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', '')); u = r[ui]
    ns = v * 1000 if u == 'usecond' else (v * 1e6 if u == 'msecond' else v)
    name = r[ki].split('(')[0][-60:]
    agg[name][0] += 1; agg[name][1] += ns; tot += ns
print(f"total {tot/1e6:.3f} ms over {sum(a[0] for a in agg.values())} launches")
for k, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{ns/1e6:8.3f} ms {100*ns/tot:5.1f}% {n:5d} x {ns/n/1e3:8.1f} us  {k}")
