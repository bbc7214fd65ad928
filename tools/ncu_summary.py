"""Summarise an ncu report (--set full) into markdown for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [launches.csv] > profiles/rN_ncu_summary.md
"""

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("Duration", "us"), ("DRAM Throughput", "%"), ("Memory Throughput", "%"), ("Compute (SM) Throughput", "%"),
    ("L1/TEX Hit Rate", "%"), ("L2 Hit Rate", "%"), ("Issue Slots Busy", "%"),
    ("Warp Cycles Per Issued Instruction", "cyc"), ("Avg. Active Threads Per Warp", ""),
    ("Executed Instructions", ""), ("Registers Per Thread", ""), ("Theoretical Occupancy", "%"),
    ("Achieved Occupancy", "%"), ("Grid Size", ""), ("Block Size", ""),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum"]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = ncu_csv(rep, "details")
    h = rows[0]
    ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
    per = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[ii], r[ki].split("(")[0].replace("<unnamed>::", ""))
        per.setdefault(key, {})
        if r[mi] not in per[key]:
            per[key][r[mi]] = r[vi]
    raw = ncu_csv(rep, "raw")
    rh, rdata = raw[0], raw[2:]
    rid = rh.index("ID")
    dram = {r[rid]: sum(float(r[rh.index(m)].replace(",", "")) for m in RAW) for r in rdata}
    units = raw[1]
    dram_unit = units[rh.index(RAW[0])]
    print(f"# ncu --set full summary: `{rep.split('/')[-1]}`\n")
    print("| ID | kernel | " + " | ".join(m for m, _ in METRICS) + f" | DRAM bytes ({dram_unit}) |")
    print("|" + "---|" * (len(METRICS) + 3))
    for (i, name), m in per.items():
        print(f"| {i} | `{name[:48]}` | " + " | ".join(m.get(k, "") for k, _ in METRICS) +
              f" | {dram.get(i, 0):.3f} |")
    if len(sys.argv) > 2:
        lr = list(csv.reader(open(sys.argv[2])))
        hi = [i for i, r in enumerate(lr) if r and r[0] == "ID"][0]
        hh, data = lr[hi], lr[hi + 1:]
        kn, mv = hh.index("Kernel Name"), hh.index("Metric Value")
        agg = collections.OrderedDict()
        for r in data:
            agg.setdefault(r[kn].split("(")[0].replace("<unnamed>::", "")[:60], []).append(
                float(r[mv].replace(",", "")))
        tot = sum(sum(v) for v in agg.values())
        print("\n## launch list (gpu__time_duration.sum, --clock-control none; cold, serialised)\n")
        print("| kernel | launches | mean ns | share |")
        print("|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.0f} | {100 * sum(v) / tot:.1f}% |")


if __name__ == "__main__":
    main()
