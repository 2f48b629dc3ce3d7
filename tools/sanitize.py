#!/usr/bin/env python
"""Small invocations of every kernel family through the C-ABI, sized for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  K1 warp rows + split GEMM (tcgen05, 2-CTA) + LR1   f16, 640 rows
  K1 row groups + decode GEMV kernels                f16, 5 rows
  K1 fp32 row-group kernel                            f32, 200 rows
  K1 fp64 MAC pass (8-bit aux codes)                  f16, 700 rows, A8
  packed 4-bit main weights (tcgen05 unpack warps)    f16, 300 rows
  MOCD absmax / rank counts / text score / top-k     f16, 3000 x 96
Exits 0 when every call returns and the device status words are clear."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
import paper_2605_19929_b200 as pkg  # noqa: E402
from paper_2605_19929_b200 import mocd_gpu, runtime  # noqa: E402


def case(seed, T, d_in, d_out, k, r_s, r_c, abits=4, dtype=np.float16):
    rng = np.random.default_rng(seed)
    tags = wl.tags_with_spans(rng, T, T // 4)
    c_t, c_v = wl.outlier_sets(rng, d_in, k)
    x = wl.make_activations(rng, T, d_in, tags, c_t, c_v, dtype=np.float32)
    layer = wl.build_split_layer(pkg, rng, wl.LayerSpec("s", d_in, d_out, k, k, r_s, r_c, abits, 4),
                                 np.max(np.abs(x), axis=0), c_t, c_v)
    g = runtime.GpuLayer(layer, runtime.device())
    xd = torch.from_numpy(x.astype(dtype)).cuda()
    td = torch.from_numpy(tags).cuda()
    y = g.run(xd, td)  # status checked (raises on a device error word)
    raw = g.run(xd, td, raw=True)
    torch.cuda.synchronize()
    return float(y.float().abs().sum()), int(raw[0].abs().sum())


out = []
out.append(case(1, 640, 512, 384, 16, 16, 16))           # warp rows, tcgen05 split GEMM + LR1
out.append(case(2, 5, 512, 256, 16, 8, 8))               # decode: row groups + GEMV
out.append(case(3, 200, 384, 160, 8, 4, 6, dtype=np.float32))
out.append(case(4, 700, 640, 256, 32, 10, 15, abits=8))  # fp64 MAC pass
out.append(case(5, 300, 1024, 256, 16, 8, 8))            # packed 4-bit weights (<= 2048 rows)
rng = np.random.default_rng(9)
x = (rng.standard_normal((3000, 96)) * rng.uniform(0.1, 5, 96)).astype(np.float16)
tags = rng.permutation(np.array([0] * 2200 + [1] * 800, np.uint8))
part = mocd_gpu.build_partition(pkg.ActivationBatch(torch.from_numpy(x).cuda(), torch.from_numpy(tags).cuda()),
                                pkg.MocdConfig(0.05, 0.05))
torch.cuda.synchronize()
print("ok", out, len(part.c_text), len(part.c_vision))
