"""DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and SM issue utilisation per kernel launch from ncu
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
        res.append((d.get("Kernel Name", ""), num("dram__bytes_read.sum") * scale + num("dram__bytes_write.sum") * scale_w,
                    num("gpu__time_duration.sum"), num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    num("inst_executed") or num("smsp__inst_executed.sum"),
                    num("sass__thread_inst_executed_true_per_opcode"),
                    num("sm__warps_active.avg.pct_of_peak_sustained_active")))
    return res


out = {}
for arg in sys.argv[1:]:
    key, spec = arg.split("=", 1)
    rep, _, rx = spec.partition(":")
    sel = [x for x in launches(rep) if not rx or re.search(rx, x[0])]
    dur = sum(x[2] for x in sel) or 1.0
    out[key] = {"bytes": sum(x[1] for x in sel), "launches": len(sel), "report": rep.rsplit("/", 1)[-1],
                # SM issue-slot utilisation (duration-weighted over the launches): the ceiling
                # of the L1-resident, issue-bound traversal
                "issue_active_pct": round(sum(x[2] * x[3] for x in sel) / dur, 2),
                # warp instructions issued per launch set (the issue roofline's numerator, divided
                # by the live launch time in bench.py), active threads per warp instruction (SIMT
                # efficiency x 32) and achieved occupancy (duration-weighted)
                "warp_inst": sum(x[4] for x in sel),
                "threads_per_inst": round(sum(x[5] for x in sel) / max(sum(x[4] for x in sel), 1.0), 2),
                "achieved_occupancy_pct": round(sum(x[2] * x[6] for x in sel) / dur, 2),
                "kernels": sorted({re.sub(r"\(.*", "", x[0]).replace("<unnamed>::", "") for x in sel})}
print(json.dumps(out, indent=1))
