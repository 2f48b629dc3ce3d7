#!/usr/bin/env python
"""Phase timeline of the prefill LR1 GEMM (needs a -DG2_TRACE build; run with
SPLITQ_TRACE_MODE=2 so only LR1 launches are traced: the last one, the MAC
first stage, is reported). python tools/lr1_phase.py [--model 3b] T..."""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import workloads as wl  # noqa: E402
import paper_2605_19929_b200 as pkg  # noqa: E402
from paper_2605_19929_b200 import runtime, _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("tokens", nargs="*", type=int, default=[4096, 8192])
ap.add_argument("--model", default="7b")
ap.add_argument("--proj", default="q")
a = ap.parse_args()
lib = _lib.load()
fn = lib.splitq_debug_gemm_trace
fn.restype = C.c_int
fn.argtypes = [C.c_void_p]
dev = torch.device("cuda", 0)
shape = wl.QWEN_3B if a.model == "3b" else wl.QWEN_7B
rng = np.random.default_rng(0)
sp = next(s for s in wl.model_specs(shape) if s.name == a.proj)
c_t, c_v = wl.outlier_sets(rng, sp.d_in, sp.k_text)
layer = wl.build_split_layer(pkg, rng, sp, np.full(sp.d_in, 4.5), c_t, c_v)
gl = runtime.GpuLayer(layer, dev)
for T in a.tokens:
    tags = torch.from_numpy(wl.tags_with_spans(rng, T, T * 5 // 32)).to(dev)
    x = torch.randn((T, sp.d_in), device=dev).half()
    y = torch.empty((T, sp.d_out), dtype=torch.float16, device=dev)
    ws = gl.workspace(T)
    for _ in range(3):
        gl.run(x, tags, y=y, check=False, ws=ws)
    torch.cuda.synchronize()
    buf = np.zeros(148 * 8, np.uint64)
    n = fn(buf.ctypes.data)
    if n == 0:
        print(f"{a.model} {a.proj} T={T}: no trace (not a -DG2_TRACE build)", flush=True)
        continue
    t = buf.reshape(148, 8)[:n].astype(np.int64)
    t0 = t[:, 0][t[:, 0] > 0].min()

    def rel(c):
        v = t[:, c][t[:, c] > 0]
        return (v - t0) / 1e3 if len(v) else np.array([-1.0])
    print(f"{a.model} {a.proj} T={T} ctas={n}: start {rel(0).min():.1f}-{rel(0).max():.1f} us, setup "
          f"{np.median(rel(1)):.1f}, first data {np.median(rel(2)):.1f}, last MMA {np.median(rel(3)):.1f}, "
          f"acc ready {np.median(rel(6)):.1f}, 1st chunk {np.median(rel(7)):.1f}, epilogue done {np.median(rel(4)):.1f} (max {rel(4).max():.1f}), "
          f"end {rel(5).max():.1f} us", flush=True)
