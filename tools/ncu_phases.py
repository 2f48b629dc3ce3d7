#!/usr/bin/env python
"""Instructions executed / stall samples between consecutive BAR.SYNC (or
other marker) instructions of a kernel's SASS, in address order."""
import csv
import subprocess
import sys

rep = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 else "BAR.SYNC"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr = None
seg = [0, 0, 0, ""]
segs = []
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
    i, s = int(r[ie]), int(r[st])
    seg[0] += i
    seg[1] += s
    seg[2] += 1
    if not seg[3] and i:
        seg[3] = r[1].strip()[:50]
    if marker in r[1]:
        segs.append(seg)
        seg = [0, 0, 0, ""]
segs.append(seg)
ti = sum(x[0] for x in segs) or 1
ts = sum(x[1] for x in segs) or 1
for k, (i, s, n, first) in enumerate(segs):
    print(f"seg {k:2d}: {n:5d} sass  {100*i/ti:5.1f}% inst  {100*s/ts:5.1f}% stall   {i:>11d}  first: {first}")
