"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name", "gpu__time_duration.sum") == "gpu__time_duration.sum":
            data.append(d)
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for d in data:
    key = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")[:70]
    us = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    agg[key][0] += 1
    agg[key][1] += us
    tot += us
print(f"{len(data)} launches, {tot / 1000:.3f} ms of kernel time (serialised, cold cache)")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{us:9.1f} us {us / tot * 100:5.1f}%  n={n:4d}  {k}")
