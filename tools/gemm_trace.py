#!/usr/bin/env python
"""Phase timeline of the split GEMM at decode sizes (needs a -DG2_TRACE build)."""
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
fn = lib.splitq_debug_gemm_trace
fn.restype = C.c_int
fn.argtypes = [C.c_void_p]
dev = torch.device("cuda", 0)
tags, inputs, layers = bench.build_workload(pkg, 64, 4, 4)
for name in sys.argv[1:] or ["q", "gate"]:
    g, sp, layer = next(t for t in layers if t[1].name == name)
    gl = runtime.GpuLayer(layer, dev)
    for B in (64, 8192):
        tg = torch.zeros(B, dtype=torch.uint8, device=dev)
        x = bench.make_input_tensor(torch, dev, B, inputs[g], np.zeros(B, np.uint8), 3)
        y = torch.empty((B, sp.d_out), dtype=torch.float16, device=dev)
        ws = gl.workspace(B)
        for _ in range(3):
            gl.run(x, tg, y=y, check=False, ws=ws)
        torch.cuda.synchronize()
        buf = np.zeros(148 * 8, np.uint64)
        n = fn(buf.ctypes.data)
        t = buf.reshape(148, 8)[:n].astype(np.int64)
        t0 = t[:, 0][t[:, 0] > 0].min()
        rel = lambda c: (t[:, c][t[:, c] > 0] - t0) / 1e3
        print(f"{name} B={B} ctas={n}: start {rel(0).min():.1f}-{rel(0).max():.1f} us, setup done "
              f"{np.median(rel(1)):.1f}, first data {np.median(rel(2)) if len(rel(2)) else -1:.1f}, "
              f"last MMA {np.median(rel(3)) if len(rel(3)) else -1:.1f}, acc ready {np.median(rel(6)):.1f}, epilogue done "
              f"{np.median(rel(4)):.1f} (max {rel(4).max():.1f}), end {rel(5).max():.1f} us", flush=True)
