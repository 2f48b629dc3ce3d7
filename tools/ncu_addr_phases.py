#!/usr/bin/env python
"""Instructions executed per kernel phase: SASS rows of an ncu source page
(--print-source cuda,sass, csv.gz) sorted by address, each attributed to the
last kernel-body line (>= BODY in FILE) seen at a lower address; phases are
line ranges given as name:first-last.
Usage: ncu_addr_phases.py SRC.csv.gz FILE BODY name:a-b ..."""
import csv
import gzip
import sys

src, fname, body = sys.argv[1], sys.argv[2], int(sys.argv[3])
phases = [(a.split(":")[0], *map(int, a.split(":")[1].split("-"))) for a in sys.argv[4:]]
rows = []
f = line = None
for r in csv.reader(gzip.open(src, "rt")):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        continue
    if r[0] and r[0].isdigit():
        line = (f, int(r[0]))
        continue
    if len(r) > 7 and r[2].startswith("0x"):
        rows.append((int(r[2], 16), line, int(r[7]), int(r[4]), r[3].strip()))
rows.sort()
# a SASS row is listed under every source line it maps to (inlining): keep
# each address once, attributed to its first-listed line inside FILE if any
seen = {}
for r in rows:
    if r[0] not in seen or (seen[r[0]][1][0] != fname and r[1][0] == fname):
        seen[r[0]] = r
rows = sorted(seen.values())
acc = {}
cur = "pre"
tot = sum(x[2] for x in rows) or 1
stot = sum(x[3] for x in rows) or 1
for addr, (fl, ln), ie, st, s in rows:
    if fl == fname and ln >= body:
        cur = next((n for n, a, b in phases if a <= ln <= b), f"L{ln}")
    a = acc.setdefault(cur, [0, 0, 0])
    a[0] += ie
    a[1] += st
    a[2] += 1
print(f"total executed {tot}, stall samples {stot}")
for k, (ie, st, n) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    if ie or st:
        print(f"{k:12s} {100*ie/tot:5.1f}% inst {100*st/stot:5.1f}% stall  {n:5d} sass  {ie}")
