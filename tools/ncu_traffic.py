"""DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per kernel launch from ncu
--set full reports -> profiles/ncu_traffic.json (read by bench.py for roofline.traffic).

    python tools/ncu_traffic.py KEY=report.ncu-rep[:kernel-regex] ... > profiles/ncu_traffic.json

Each KEY sums the matching launches of its report (e.g. the 10 kernels of one LBVH build).
"""
import csv
import io
import json
import re
import subprocess
import sys


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        def num(k):
            v = d.get(k, "0").replace(",", "")
            try:
                return float(v)
            except ValueError:
                return 0.0
        unit = rows[1][h.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in h else "byte"
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        unit_w = rows[1][h.index("dram__bytes_write.sum")] if "dram__bytes_write.sum" in h else "byte"
        scale_w = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit_w, 1)
        res.append((d.get("Kernel Name", ""), num("dram__bytes_read.sum") * scale + num("dram__bytes_write.sum") * scale_w))
    return res


out = {}
for arg in sys.argv[1:]:
    key, spec = arg.split("=", 1)
    rep, _, rx = spec.partition(":")
    sel = [(k, b) for k, b in launches(rep) if not rx or re.search(rx, k)]
    out[key] = {"bytes": sum(b for _, b in sel), "launches": len(sel), "report": rep.rsplit("/", 1)[-1],
                "kernels": sorted({re.sub(r"\(.*", "", k).replace("<unnamed>::", "") for k, _ in sel})}
print(json.dumps(out, indent=1))
