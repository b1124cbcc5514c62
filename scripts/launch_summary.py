"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel.

--last-eval keeps only the launches of the final kafmm_eval (from the last
k_gather on), i.e. one step of the hot path.
"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) > h.index('Metric Value')]
ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
if '--last-eval' in sys.argv:
    last = max(i for i, r in enumerate(data) if 'k_gather' in r[ki])
    data = data[last:]
scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0, 's': 1e3, 'second': 1e3}
agg = collections.OrderedDict(); n = collections.Counter()
for r in data:
    name = r[ki].split('(')[0]
    v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    agg[name] = agg.get(name, 0) + v; n[name] += 1
tot = sum(agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k[:60]:60s} {n[k]:8d} {v:10.3f} {100 * v / tot:6.2f}%")
print(f"{'total':60s} {sum(n.values()):8d} {tot:10.3f}")
