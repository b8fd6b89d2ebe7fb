"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: time per kernel (ms) and share."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        ms = v / 1e6 if unit in ("ns", "nsecond") else v / 1e3 if unit in ("us", "usecond") else v
        name = d["Kernel Name"].split("(")[0][:70]
        agg.setdefault(name, [0.0, 0])
        agg[name][0] += ms
        agg[name][1] += 1
tot = sum(v[0] for v in agg.values())
for k, (ms, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{ms:9.3f} ms {100 * ms / tot:5.1f}%  x{c:<3d} {k}")
print(f"{tot:9.3f} ms total")
