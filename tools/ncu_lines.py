#!/usr/bin/env python
"""Per-CUDA-line instruction counts and stall samples from an ncu report
(ncu -i REP --page source --csv --print-source cuda,sass)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
f = "?"
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0] or not r[0].isdigit():
        continue
    try:
        stall = int(r[4]); ie = int(r[7])
    except ValueError:
        continue
    rows.append((f, int(r[0]), r[1].strip()[:90], stall, ie))
tot_i = sum(x[4] for x in rows) or 1
tot_s = sum(x[3] for x in rows) or 1
print(f"total inst {tot_i}  stall samples {tot_s}")
print("--- by instructions")
for x in sorted(rows, key=lambda x: -x[4])[:top]:
    print(f"{x[0]}:{x[1]:4d} {100*x[4]/tot_i:5.1f}% inst {100*x[3]/tot_s:5.1f}% stall | {x[2]}")
print("--- by stall samples")
for x in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{x[0]}:{x[1]:4d} {100*x[4]/tot_i:5.1f}% inst {100*x[3]/tot_s:5.1f}% stall | {x[2]}")
