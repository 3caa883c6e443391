#!/usr/bin/env python
"""Groups an ncu launch list (`--metrics gpu__time_duration.sum --csv`) by kernel: total device time, share, launches.
usage: launch_summary.py launches.csv"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]; col = {h: i for i, h in enumerate(hdr)}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) != len(hdr) or r[col["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[col["Metric Value"]]); u = r[col["Metric Unit"]]
    v = v / 1e3 if u in ("usecond", "us") else v / 1e6 if u in ("nsecond", "ns") else v * 1e3 if u in ("second", "s") else v
    agg[r[col["Kernel Name"]]][0] += 1; agg[r[col["Kernel Name"]]][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{sum(v[0] for v in agg.values())} launches, {tot:.2f} ms of device time (cold-cache, serialised: compare SHARES)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1]:10.2f} ms {100 * v[1] / tot:5.1f}%  x{v[0]:3d}  {k[:140]}")
