"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) by kernel: count, total, share."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); gi = h.index('Grid Size')
c, t = Counter(), Counter()
for r in rows[hdr + 1:]:
    name = r[ki].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '')[:60]
    c[name] += 1; t[name] += float(r[vi].replace(',', ''))
tot = sum(t.values())
print(f"{len(rows)-hdr-1} launches, {tot/1e6:.3f} ms total (ncu: cold-cache, serialised)")
for k, v in t.most_common():
    print(f"{v/1e6:9.3f} ms {100*v/tot:5.1f}% {c[k]:5d}x  avg {v/c[k]/1e3:8.1f} us  {k}")
