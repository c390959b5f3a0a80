"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel and grid."""
import collections
import csv
import re
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
data = rows[hi + 1:]
ki, mi, gi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size'), h.index('Metric Unit')
tot = collections.defaultdict(float)
cnt = collections.Counter()
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
for r in data:
    v = float(r[mi].replace(',', '')) * scale.get(r[ui], 1e-3)
    name = r[ki].replace('void ', '')
    m = re.match(r'([\w:]+)<([^>]*)>', name)
    key = (m.group(0) if m else name.split('(')[0], r[gi])
    tot[key] += v
    cnt[key] += 1
T = sum(tot.values())
print(f"# total {T / 1000:.2f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:9.1f} us {100 * v / T:5.1f}% n={cnt[k]:5d} avg={v / cnt[k]:8.2f}us  {k[0][:44]:44s} grid={k[1]}")
