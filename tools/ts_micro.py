#!/usr/bin/env python
"""Time the MOCD text-score kernel (exact 1-D k-means per candidate channel)
on synthetic rank counts: --n-cand candidates (the rank denominator),
--n-text text rows, --channels scored (one CTA each)."""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_19929_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n-cand", type=int, default=18755)
ap.add_argument("--n-text", type=int, default=196608)
ap.add_argument("--channels", type=int, default=592)
ap.add_argument("--k", type=int, default=3)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
# iid rows: each column's rank counts are ~uniform over 1..n_cand
counts_t = torch.randint(1, a.n_cand + 1, (a.channels, a.n_text), device="cuda", generator=g,
                         dtype=torch.int32).to(torch.int16)
scores = torch.empty(a.channels, dtype=torch.float64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def run():
    _lib.check(lib.splitq_mocd_text_score(counts_t.data_ptr(), counts_t.stride(0), a.n_cand, a.n_text,
                                          a.k, 50, 0, a.channels, scores.data_ptr(), st))


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    run()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / a.iters
print(f"text_score {a.channels} channels x {a.n_text} rows (n_cand {a.n_cand}, k {a.k}): {ms:.2f} ms, "
      f"{ms / a.channels * 1e3:.1f} us per channel; checksum {float(scores.sum()):.17g}")
