"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][:60]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
allt = sum(tot.values())
print(f"{len(data)} launches, {allt / 1e3:.3f} ms total")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us {100 * v / allt:5.1f}%  x{cnt[k]:3d}  {v / cnt[k]:9.1f} us/launch  {k}")
