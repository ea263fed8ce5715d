"""Summarize an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
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
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(list)
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for d in data:
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("(anonymous namespace)::", "")
    agg[name[:80]].append(float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]])
tot = sum(sum(v) for v in agg.values())
print(f"{len(data)} launches, {tot/1e3:.3f} ms total")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v)/1e3:9.3f} ms {100*sum(v)/tot:5.1f}%  n={len(v):5d}  avg={sum(v)/len(v):9.1f} us  max={max(v):9.1f} us  {k}")
