#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run where ncu is available).

  ncu_summary.py launches <launches.csv> <out.json>
      per-kernel launch counts, total / mean time and share of the run from
      an `ncu --metrics gpu__time_duration.sum --csv` launch list
  ncu_summary.py full <report.ncu-rep> <out.json>
      the key sections (duration, throughput, IPC, occupancy, DRAM bytes,
      tensor-pipe activity, stall reasons) of every kernel in a
      `ncu --set full` report
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    seq = []
    for r in rows[hi + 1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
        seq.append((name, v / 1e3))
    tot = sum(v for _, v in agg.values())
    res = {"source": path, "unit": "us", "total_us": tot / 1e3,
           "kernels": [{"kernel": k, "launches": n, "total_us": v / 1e3, "mean_us": v / n / 1e3,
                        "share": v / tot} for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])],
           "sequence_us": seq}
    json.dump(res, open(out, "w"), indent=1)


WANT = {
    "Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
    "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
    "Achieved Active Warps Per SM", "Theoretical Occupancy", "Executed Instructions",
    "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size", "L1/TEX Hit Rate", "L2 Hit Rate",
    "Dynamic Shared Memory Per Block",
}
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
       "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active")


def full(path, out):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    kernels = defaultdict(dict)
    r = list(csv.reader(io.StringIO(det))) or [[]]
    h = r[0]
    for row in (r[1:] if "Metric Name" in h else []):
        m = row[h.index("Metric Name")]
        if m in WANT:
            key = f'{row[h.index("ID")]}:{row[h.index("Kernel Name")].split("(")[0]}'
            kernels[key][m] = f'{row[h.index("Metric Value")]} {row[h.index("Metric Unit")]}'.strip()
    r = list(csv.reader(io.StringIO(raw))) or [[]]
    h = r[0]
    units = r[1] if len(r) > 1 else []
    for row in (r[2:] if "ID" in h else []):
        key = f'{row[h.index("ID")]}:{row[h.index("Kernel Name")].split("(")[0]}'
        for i, name in enumerate(h):
            base = name.split(".", 1)[1] if name.startswith("TPC.") else name
            if base in RAW or any(t in name for t in ("pipe_tensor", "mem_tensor_cycles")):
                if name.endswith(("pct_of_peak_sustained_elapsed", "pct_of_peak_sustained_active", ".sum")):
                    kernels[key][name] = row[i]
                    if i < len(units) and units[i]:
                        kernels[key][name + ".unit"] = units[i]
        stalls = {}
        for i, name in enumerate(h):
            if name.startswith("smsp__average_warps_issue_stalled") and name.endswith("per_issue_active.ratio"):
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v >= 0.2:
                    stalls[name.split("stalled_")[1].split("_per_issue")[0]] = round(v, 3)
        kernels[key]["stall_cycles_per_issue"] = stalls
    json.dump({"source": path, "kernels": kernels}, open(out, "w"), indent=1)


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
