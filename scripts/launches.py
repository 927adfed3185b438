"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = re.sub(r"\(.*", "", d["Kernel Name"])[:60]
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
            agg[k][0] += 1
            agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:10.1f} us {v[0]:5d} {v[1] / max(v[0], 1):8.2f} us/launch {100 * v[1] / tot:5.1f}%  {k}")
print(f"total {tot:.1f} us")
