#!/usr/bin/env python
"""Phase clocks of one K1 row at decode sizes (needs a -DKW_TRACE build):
cycles spent between the KW_STAMP points of k1w.cuh for CTA 0's first row."""
import ctypes as C
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_19929_b200 as pkg  # noqa: E402
from paper_2605_19929_b200 import runtime, _lib  # noqa: E402
lib = _lib.load()
fn = lib.splitq_debug_k1_trace
fn.restype = C.c_int
fn.argtypes = [C.c_void_p]
NAMES = ["passA", "site0", "band+site1", "params", "outlier codes", "passE", "allx site2", "fixupE",
         "FL site3", "MAC band", "site4", "MAC params", "passG", "site5", "fixupG"]
dev = torch.device("cuda", 0)
tags, inputs, layers = bench.build_workload(pkg, 64, 4, 4)
for name in sys.argv[1:] or ["q", "down"]:
    g, sp, layer = next(t for t in layers if t[1].name == name)
    gl = runtime.GpuLayer(layer, dev)
    for B in (1, 8):
        tg = torch.zeros(B, dtype=torch.uint8, device=dev)
        x = bench.make_input_tensor(torch, dev, B, inputs[g], np.zeros(B, np.uint8), 3)
        y = torch.empty((B, sp.d_out), dtype=torch.float16, device=dev)
        ws = gl.workspace(B)
        acc = np.zeros(16)
        for it in range(13):
            gl.run(x, tg, y=y, check=False, ws=ws)
            buf = np.zeros(16, np.uint64)
            fn(buf.ctypes.data)
            if it >= 3:
                acc += buf.astype(np.float64)
        t = acc / 10
        d = np.diff(t)
        print(name, B, "total", int(t[15] - t[0]), "cycles;",
              ", ".join(f"{n} {int(v)}" for n, v in zip(NAMES, d)), flush=True)
