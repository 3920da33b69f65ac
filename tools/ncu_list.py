"""Summarise an ncu --csv launch list (gpu__time_duration + optional dram bytes) per launch."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
k = OrderedDict()
for r in rows[start + 1:]:
    k.setdefault((r[ix["ID"]], r[ix["Kernel Name"]][:60]), {})[r[ix["Metric Name"]]] = r[ix["Metric Value"]]
f = lambda v: float(v.replace(",", ""))
for (i, n), m in k.items():
    t = f(m["gpu__time_duration.sum"]) / 1e3
    rd = f(m.get("dram__bytes_read.sum", "0")) / 1e6
    wr = f(m.get("dram__bytes_write.sum", "0")) / 1e6
    print(f"{i:>4} {n:<60} {t:9.2f} us  rd {rd:8.1f} MB  wr {wr:7.1f} MB  {(rd + wr) / max(t, 1e-9) * 1e-3:6.2f} TB/s")
