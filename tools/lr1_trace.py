#!/usr/bin/env python
"""Phase timeline of one prefill GEMM launch (needs a -DG2_TRACE build; set
SPLITQ_TRACE_MODE=2 for the low-rank first stage, 0 for the split GEMM)."""
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
T = 65536
tags, inputs, layers = bench.build_workload(pkg, T, 4, 4)
for name in sys.argv[1:] or ["q"]:
    g, sp, layer = next(t for t in layers if t[1].name == name)
    gl = runtime.GpuLayer(layer, dev)
    x = bench.make_input_tensor(torch, dev, T, inputs[g], tags, 3)
    tg = torch.from_numpy(tags).to(dev)
    y = torch.empty((T, sp.d_out), dtype=torch.float16, device=dev)
    ws = gl.workspace(T)
    for _ in range(3):
        gl.run(x, tg, y=y, check=False, ws=ws)
    torch.cuda.synchronize()
    buf = np.zeros(148 * 8, np.uint64)
    n = fn(buf.ctypes.data)
    t = buf.reshape(148, 8)[:n].astype(np.int64)
    t0 = t[:, 0][t[:, 0] > 0].min()
    rel = lambda c: (t[:, c][t[:, c] > 0] - t0) / 1e3
    print(f"{name} mode={os.environ.get('SPLITQ_TRACE_MODE')} ctas={n}: start {rel(0).min():.1f}-{rel(0).max():.1f}, "
          f"setup {np.median(rel(1)):.1f}, first data {np.median(rel(2)):.1f}, acc ready {np.median(rel(6)):.1f}, "
          f"last MMA {np.median(rel(3)):.1f} (max {rel(3).max():.1f}), epilogue done {np.median(rel(4)):.1f} "
          f"(max {rel(4).max():.1f}), end {rel(5).max():.1f} us", flush=True)
