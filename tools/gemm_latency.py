#!/usr/bin/env python
"""Back-to-back raw int8 GEMM launches (splitq_gemm_i8) at decode shapes:
per-launch device time, to separate fixed kernel cost from data movement."""
import ctypes as C
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_19929_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
shapes = [(8192, 128, 3584), (8192, 96, 3584), (8192, 256, 3584), (8192, 3584, 3584), (16384, 3584, 3584),
          (64, 3584, 3584), (64, 512, 3584)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for (m, n, k) in shapes:
    a = torch.randint(-8, 8, (m, k), dtype=torch.int8, device=dev)
    b = torch.randint(-8, 8, (n, k), dtype=torch.int8, device=dev)
    c = torch.empty((m, n), dtype=torch.int32, device=dev)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    def run():
        _lib.check(lib.splitq_gemm_i8(a.data_ptr(), k, 1, b.data_ptr(), k, c.data_ptr(), n, m, n, k, st))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        run()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    print(f"raw GEMM {m}x{n}x{k}: {us:.1f} us/launch, {2*m*n*k/us/1e6:.0f} TOPS, weights {n*k/us/1e3:.0f} GB/s", flush=True)
