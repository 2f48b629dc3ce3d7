#!/usr/bin/env python
"""Print the SASS (with executed counts) of one BAR.SYNC-delimited segment."""
import csv
import subprocess
import sys

rep, want = sys.argv[1], int(sys.argv[2])
minc = int(sys.argv[3]) if len(sys.argv) > 3 else 1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr = None
k = 0
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "Address":
        hdr = r
        ie = hdr.index("Instructions Executed")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r[0].startswith("0x"):
        continue
    if k == want and int(r[ie]) >= minc:
        print(f"{int(r[ie]):>10d} {int(r[st]):>6d}  {r[1].strip()}")
    if "BAR.SYNC" in r[1]:
        k += 1
