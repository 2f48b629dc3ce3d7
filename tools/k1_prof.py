#!/usr/bin/env python
"""One 7B projection at config-3 shapes through GpuLayer.run: a short, ncu-friendly
K1 (+ LR1 + split GEMM) workload. --proj q|down, --tokens N, --iters K."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import workloads as wl  # noqa: E402
import paper_2605_19929_b200 as pkg  # noqa: E402
from paper_2605_19929_b200 import runtime  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--proj", default="q")
ap.add_argument("--tokens", type=int, default=65536)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--abits", type=int, default=4)
a = ap.parse_args()
rng = np.random.default_rng(0)
shape = wl.QWEN_7B
sp = next(s for s in wl.model_specs(shape, abits=a.abits) if s.name == a.proj)
c_t, c_v = wl.outlier_sets(rng, sp.d_in, sp.k_text)
spec_in = dict(c_t=c_t, c_v=c_v, d_in=sp.d_in, scales_t=rng.uniform(30, 100, len(c_t)),
               scales_v=rng.uniform(30, 100, len(c_v)))
col_max = np.full(sp.d_in, 4.5)
col_max[c_t] = 4.5 * spec_in["scales_t"]
col_max[c_v] = 4.5 * spec_in["scales_v"]
layer = wl.build_split_layer(pkg, rng, sp, col_max, c_t, c_v)
tags = np.concatenate([wl.tags_with_spans(rng, 8192, 1280) for _ in range(max(1, a.tokens // 8192))])[:a.tokens]
dev = torch.device("cuda", 0)
x = bench.make_input_tensor(torch, dev, a.tokens, spec_in, tags, 1)
t = torch.from_numpy(tags).to(dev)
g = runtime.packed(layer)
ws = g.workspace(a.tokens)
y = torch.empty((a.tokens, sp.d_out), dtype=torch.float16, device=dev)
for _ in range(2):  # warm-up (first-call set-up, attributes, tensor maps)
    g.run(x, t, y=y, ws=ws, profile=True)
torch.cuda.synchronize()
g.profile_read()
for _ in range(a.iters):
    g.run(x, t, y=y, ws=ws, profile=True)
torch.cuda.synchronize()
ms, calls = g.profile_read()
print({"proj": a.proj, "tokens": a.tokens, "stage_ms": [m / calls for m in ms]})
