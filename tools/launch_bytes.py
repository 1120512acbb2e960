"""Per-launch device time, DRAM bytes and GB/s from an ncu --csv launch list."""
import csv
import sys
from collections import OrderedDict

SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
      "msecond": 1.0, "nsecond": 1e-6}
recs = OrderedDict()
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"].split("(")[0].replace("void ", "").replace("bmmgpu::<unnamed>::", ""))
        recs.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SC.get(
            d["Metric Unit"], 1)
for (i, k), m in recs.items():
    t = m.get("gpu__time_duration.sum", 0)
    b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    print(f"{i:>4} {k[:44]:44s} {t:9.3f} ms {b / 1e9:8.2f} GB {b / 1e9 / max(t, 1e-9):8.1f} GB/s")
