"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (development aid)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg.setdefault(r[ki][:80], []).append(float(r[vi].replace(',', '')))
for k, v in agg.items():
    print(f"{len(v):3d} x {sum(v)/len(v)/1e3:10.1f} us  {k}")
