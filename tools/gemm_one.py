#!/usr/bin/env python
"""One split-linear forward of a Qwen2.5-VL-7B projection at 65,536 tokens
(W4A4), repeated --reps times: the target for an ncu capture of the
split GEMM at the bench's shape (python tools/gemm_one.py q)."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
import paper_2605_19929_b200 as pkg  # noqa: E402
from paper_2605_19929_b200 import runtime  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("proj", nargs="?", default="q")
ap.add_argument("--tokens", type=int, default=65536)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
rng = np.random.default_rng(0)
sp = next(s for s in wl.model_specs(wl.QWEN_7B) if s.name == args.proj)
c_t, c_v = wl.outlier_sets(rng, sp.d_in, sp.k_text)
layer = wl.build_split_layer(pkg, rng, sp, np.full(sp.d_in, 4.5), c_t, c_v)
g = runtime.GpuLayer(layer)
T = args.tokens
tags = torch.from_numpy(wl.tags_with_spans(rng, T, T * 5 // 32)).cuda()
x = torch.randn((T, sp.d_in), device="cuda").half()
y = torch.empty((T, sp.d_out), device="cuda", dtype=torch.float16)
ws = g.workspace(T)
for _ in range(args.reps):
    g.run(x, tags, y=y, ws=ws, check=False)
torch.cuda.synchronize()
print("ok", args.proj, T)
