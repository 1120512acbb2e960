"""Aggregate an ncu --metrics gpu__time_duration.sum launch list by kernel name."""
import csv
import sys
from collections import OrderedDict

agg = OrderedDict()
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("bmmgpu::<unnamed>::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        ms = v / 1e6 if unit == "ns" else v / 1e3 if unit == "us" else v if unit == "ms" else v * 1e3
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + ms)
tot = sum(t for _, t in agg.values())
for k, (c, t) in agg.items():
    print(f"{k[:60]:60s} {c:5d} {t:10.3f} ms {100*t/tot:5.1f}%")
print(f"{'total':60s} {sum(c for c,_ in agg.values()):5d} {tot:10.3f} ms")
