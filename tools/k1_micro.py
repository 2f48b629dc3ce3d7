#!/usr/bin/env python
"""Time the K1 per-token quantizer alone (splitq_quantize_rows) on a
[rows x cols] fp16 matrix; prints GB/s against the HBM roofline."""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_19929_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=65536)
ap.add_argument("--cols", type=int, default=3520)
ap.add_argument("--bits", type=int, default=4)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
lib = _lib.load()
x = torch.randn((a.rows, a.cols), device="cuda", dtype=torch.float16)
ld = (a.cols + 15) // 16 * 16
codes = torch.empty((a.rows, ld), dtype=torch.int8, device="cuda")
s = torch.empty(a.rows, dtype=torch.float64, device="cuda")
z = torch.empty(a.rows, dtype=torch.int32, device="cuda")
st = torch.zeros(4, dtype=torch.int32, device="cuda")
cen = C.c_int32()
spec = _lib.QSpec(a.bits, 0)
stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def run():
    _lib.check(lib.splitq_quantize_rows(x.data_ptr(), _lib.F16, a.cols, a.rows, a.cols, spec,
                                        codes.data_ptr(), ld, s.data_ptr(), z.data_ptr(),
                                        st.data_ptr(), C.byref(cen), stream))


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    run()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / a.iters
byts = a.rows * a.cols * 2 + a.rows * ld
print(f"K1 quantize_rows {a.rows}x{a.cols}: {ms*1e3:.1f} us, {byts/ms/1e6:.0f} GB/s")
