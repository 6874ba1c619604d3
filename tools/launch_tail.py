"""Summarise the kernels after the last gpu_sleep marker in an ncu launch CSV."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
recs = []
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', '')); u = r[ui]
    us = {'nsecond': v / 1e3, 'ns': v / 1e3, 'usecond': v, 'us': v, 'msecond': v * 1e3, 'ms': v * 1e3}.get(u, v / 1e3)
    recs.append((r[ki], us))
last = max(i for i, (k, _) in enumerate(recs) if 'sleep' in k)
tail = recs[last + 1:]
agg = collections.defaultdict(lambda: [0, 0.0])
for k, us in tail:
    name = k.split('(')[0][-70:]
    agg[name][0] += 1; agg[name][1] += us
tot = sum(a[1] for a in agg.values())
print(f"{len(tail)} launches, sum {tot/1e3:.3f} ms")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{us/1e3:8.3f} ms {100*us/tot:5.1f}% {n:5d} x {us/n:8.1f} us  {k}")
