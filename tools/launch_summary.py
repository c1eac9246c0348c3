"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', '')); v *= {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}.get(r[ui], 1.0)
    name = r[ki].split('(')[0]; agg[name][0] += 1; agg[name][1] += v; tot += v
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%-46s %5d %11.1f us %6.1f%%" % (k[:46], c, v, 100 * v / tot))
print("total %.1f us" % tot)
