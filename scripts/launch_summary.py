"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel
launches, total and share."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
d = collections.OrderedDict(); tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', ''))
    d.setdefault(r[ki][:80], [0, 0.0])
    d[r[ki][:80]][0] += 1; d[r[ki][:80]][1] += v; tot += v
for k, (c, v) in sorted(d.items(), key=lambda x: -x[1][1]):
    print(f"{c:5d} {v/1e6:9.3f} ms {100*v/tot:5.1f}%  {k}")
print(f"total {tot/1e6:.3f} ms")
