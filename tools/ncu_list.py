"""Print an ncu --csv launch list (gpu__time_duration, dram bytes) compactly:
    python tools/ncu_list.py file.csv [--tide]"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
ik, im, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
launches = OrderedDict()
for r in rows[1:]:
    if len(r) <= iv:
        continue
    e = launches.setdefault(r[iid], {"k": r[ik]})
    e[r[im]] = r[iv]
only_tide = "--tide" in sys.argv
for i, e in launches.items():
    if only_tide and "tide" not in e["k"]:
        continue
    t = float(e.get("gpu__time_duration.sum", "0").replace(",", ""))
    b = float(e.get("dram__bytes_read.sum", "0").replace(",", ""))
    print(f"{i:>4} {t/1000:9.2f} us {b/1e6:9.2f} MB  {e['k'][:90]}")
