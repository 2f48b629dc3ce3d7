#!/usr/bin/env python
"""One 7B projection at decode batch sizes: stage times (K1, LR1s, split
GEMM) with packed and int8 weights. Quick iteration aid for the decode path."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2605_19929_b200 as pkg  # noqa: E402
from paper_2605_19929_b200 import runtime  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--proj", default="q")
ap.add_argument("--batches", default="1,16,64")
ap.add_argument("--iters", type=int, default=30)
a = ap.parse_args()
dev = torch.device("cuda", 0)
tags, inputs, layers = bench.build_workload(pkg, 64, 4, 4)
g, sp, layer = next(t for t in layers if t[1].name == a.proj)
gl = runtime.GpuLayer(layer, dev)
for B in (int(b) for b in a.batches.split(",")):
    tg = torch.zeros(B, dtype=torch.uint8, device=dev)
    x = bench.make_input_tensor(torch, dev, B, inputs[g], np.zeros(B, np.uint8), 3)
    y = torch.empty((B, sp.d_out), dtype=torch.float16, device=dev)
    ws = gl.workspace(B)
    for unpacked in (False, True):
        for _ in range(3):
            gl.run(x, tg, y=y, check=False, ws=ws, unpacked=unpacked)
        gl.profile_read()
        for _ in range(a.iters):
            gl.run(x, tg, y=y, check=False, ws=ws, profile=True, unpacked=unpacked)
        st, calls = gl.profile_read()
        print(f"{a.proj} B={B:3d} {'int8  ' if unpacked else 'packed'}: K1 {st[0]/calls*1e3:7.1f} us  "
              f"LR1 {st[1]/calls*1e3:7.1f} us  GEMM {st[2]/calls*1e3:7.1f} us", flush=True)
