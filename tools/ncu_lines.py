"""Aggregate an ncu report's warp-stall samples per CUDA source line (needs -lineinfo and
--import-source on): python tools/ncu_lines.py report.ncu-rep [top]
Samples of inlined code are attributed to the file/line of the inlined statement."""
import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
agg = defaultdict(lambda: [0.0, 0.0, ""])
fname, hdr = "?", None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r and r[0] == "Line No":
        hdr = r
        i_st = hdr.index("Warp Stall Sampling (All Samples)")
        i_ex = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    try:
        agg[key][0] += float(r[i_st] or 0)
        agg[key][1] += float(r[i_ex] or 0)
    except ValueError:
        continue
    if not agg[key][2]:
        agg[key][2] = r[1].strip()
tot = sum(v[0] for v in agg.values()) or 1
print(f"total samples {tot:.0f}")
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:6.2f}%  {f}:{ln:<5} ex={v[1]:.3g}  {v[2][:100]}")
