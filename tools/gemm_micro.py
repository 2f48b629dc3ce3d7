#!/usr/bin/env python
"""Time one 7B projection (split-linear forward) in isolation: per-stage
device times and the split GEMM's TOPS. --proj q|k|v|o|gate|up|down."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_19929_b200 as pkg  # noqa: E402
import workloads as wl  # noqa: E402
from paper_2605_19929_b200 import runtime  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--proj", default="q")
ap.add_argument("--tokens", type=int, default=16384)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--abits", type=int, default=4)
a = ap.parse_args()
rng = np.random.default_rng(0)
spec = next(s for s in wl.model_specs(wl.QWEN_7B, abits=a.abits) if s.name == a.proj)
c_t, c_v = wl.outlier_sets(rng, spec.d_in, spec.k_text)
col_max = np.full(spec.d_in, 4.5)
col_max[c_t] = 200.0
col_max[c_v] = 200.0
layer = wl.build_split_layer(pkg, rng, spec, col_max, c_t, c_v)
g = runtime.GpuLayer(layer)
tags = torch.from_numpy(wl.tags_with_spans(rng, a.tokens, a.tokens * 5 // 32)).cuda()
x = torch.randn((a.tokens, spec.d_in), device="cuda").half()
y = torch.empty((a.tokens, spec.d_out), device="cuda", dtype=torch.float16)
ws = g.workspace(a.tokens)
for _ in range(3):
    g.run(x, tags, y=y, ws=ws, check=False)
g.run(x, tags, y=y, ws=ws, check=True)
g.profile_read()
for _ in range(a.iters):
    g.run(x, tags, y=y, ws=ws, check=False, profile=True)
ms, calls = g.profile_read()
ops = 2.0 * a.tokens * spec.d_in * spec.d_out
print(f"{a.proj} T={a.tokens}: quant {ms[0]/calls*1e3:.1f} us, lr1 {ms[1]/calls*1e3:.1f} us, "
      f"gemm {ms[2]/calls*1e3:.1f} us = {ops/(ms[2]/calls*1e-3)/1e12:.0f} TOPS")
