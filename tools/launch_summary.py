"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
ui = hdr.index('Metric Unit') if 'Metric Unit' in hdr else None
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '').replace('cake_dev::', '')
    v = float(r[vi].replace(',', ''))
    unit = r[ui] if ui is not None else 'nsecond'
    v *= {'nsecond': 1, 'usecond': 1e3, 'msecond': 1e6}.get(unit, 1)
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:48]:48s} {cnt[k]:6d} {v / 1e6:9.2f} ms {100 * v / s:5.1f}%  avg {v / cnt[k] / 1e3:8.2f} us")
print(f"total kernel time {s / 1e6:.2f} ms")
