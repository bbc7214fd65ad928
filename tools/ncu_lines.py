"""Top CUDA source lines of one kernel in an ncu report (--import-source, -lineinfo) by
warp-stall samples, with executed warp instructions per line.

    python tools/ncu_lines.py rep.ncu-rep <kernel-regex> [top] [launch-skip]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kern, "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
data = []
fname = ""
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        samp = float(r[4] or 0)
        inst = float(r[7] or 0)
        if samp or inst:
            data.append((samp, inst, fname, r[0], r[1]))
tot = sum(d[0] for d in data) or 1
toti = sum(d[1] for d in data) or 1
print(f"total stall samples {tot:.0f}, warp instructions {toti:.0f}")
for s, i, f, ln, src in sorted(data, key=lambda d: -d[0])[:top]:
    print(f"{100*s/tot:5.1f}% smp {100*i/toti:5.1f}% inst  {f}:{ln:<5} {src.strip()[:100]}")
