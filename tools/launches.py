"""Print an ncu --metrics gpu__time_duration.sum CSV launch list as 'id kernel us'."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        name = d["Kernel Name"].replace("<unnamed>::", "").split("(")[0][:70]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        us = v / 1000 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1000)
        print(f"{d['ID']:>4} {name:<70} {us:9.2f} us")
