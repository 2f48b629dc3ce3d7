#!/usr/bin/env python
"""Measure the dense INT8 tensor peak of this B200 the way MEASURED_PEAKS.json
measures bf16: an 8192^3 cuBLASLt int8 GEMM (torch._int_mm), best of 10
(burst) and back to back for 4 s (sustained). Also times the repo's own raw
tcgen05 GEMM (splitq_gemm_i8) on the same shape. Writes profiles/int8_peak.json.
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, n):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n


def main():
    n = 8192
    a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
    ops = 2.0 * n ** 3
    out = {"shape": [n, n, n], "how": "torch._int_mm int8 8192^3 (cuBLASLt): best of 10 single "
                                       "launches (burst) and back-to-back for 4 s (sustained)"}
    bt = b.t()
    f = lambda: torch._int_mm(a, bt)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    best = min(timeit(f, 1) for _ in range(10))
    out["int8_tops"] = ops / (best * 1e-3) / 1e12
    t0 = time.time()
    iters, total = 0, 0.0
    while time.time() - t0 < 4.0:
        total += timeit(f, 10) * 10
        iters += 10
    out["int8_tops_sustained"] = ops * iters / (total * 1e-3) / 1e12
    # the repo's own kernel
    from paper_2605_19929_b200 import _lib
    lib = _lib.load()
    c = torch.empty((n, n), dtype=torch.int32, device="cuda")
    g = lambda: _lib.check(lib.splitq_gemm_i8(a.data_ptr(), n, 1, b.data_ptr(), n, c.data_ptr(), n,  # noqa: E731
                                               n, n, n, None))
    for _ in range(3):
        g()
    torch.cuda.synchronize()
    best = min(timeit(g, 1) for _ in range(10))
    out["splitq_gemm_i8_tops"] = ops / (best * 1e-3) / 1e12
    t0 = time.time()
    iters, total = 0, 0.0
    while time.time() - t0 < 4.0:
        total += timeit(g, 10) * 10
        iters += 10
    out["splitq_gemm_i8_tops_sustained"] = ops * iters / (total * 1e-3) / 1e12
    ref = torch._int_mm(a, bt)
    out["splitq_matches_cublas"] = bool(torch.equal(ref, c))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "int8_peak.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
