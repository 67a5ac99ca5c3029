"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "ID")
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    name = d["Kernel Name"].split("(")[0].replace("void ", "")[:72]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
print(f"{len(data)} launches, {tot/1e3:.2f} ms total")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{us/1e3:9.3f} ms {100*us/tot:5.1f}%  n={n:4d}  {k}")
