"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --csv) by kernel name: launches, total time, share, DRAM GB."""
import csv
import sys
from collections import OrderedDict

SCALE_T = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
SCALE_B = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}

agg = OrderedDict()  # name -> [launches, ms, dram GB]
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("bmmgpu::<unnamed>::", "")
    name = name.replace("<unnamed>::", "")
    v = float(d["Metric Value"].replace(",", ""))
    unit, metric = d["Metric Unit"], d.get("Metric Name", "gpu__time_duration.sum")
    a = agg.setdefault(name, [0, 0.0, 0.0])
    if metric == "gpu__time_duration.sum":
        a[0] += 1
        a[1] += v * SCALE_T.get(unit, 1e-6)
    elif metric.startswith("dram__bytes"):
        a[2] += v * SCALE_B.get(unit, 1e-9)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'time':>13s} {'share':>6s} {'DRAM':>10s}")
for k, (c, t, gb) in agg.items():
    print(f"{k[:60]:60s} {c:8d} {t:10.3f} ms {100 * t / tot:5.1f}% {gb:7.2f} GB")
print(f"{'total':60s} {sum(a[0] for a in agg.values()):8d} {tot:10.3f} ms")
