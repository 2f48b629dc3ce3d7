#!/usr/bin/env python
"""Split GEMM ablations on the 7B prefill shapes (65,536 tokens): cuBLASLt
int8 (torch._int_mm) vs the repo's raw tcgen05 GEMM (splitq_gemm_i8) vs the
split-linear forward's GEMM stage with and without the fp16 aux branch, at
the default and forced tile widths (SPLITQ_TILE_N). Prints TOPS per line."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
import paper_2605_19929_b200 as pkg  # noqa: E402
from paper_2605_19929_b200 import _lib, runtime  # noqa: E402

lib = _lib.load()


def best_ms(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(n):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        out.append(s.elapsed_time(e))
    return min(out)


T = 65536
for name, M, N, K in (("q", T, 3584, 3584), ("gate", T, 18944, 3584), ("down", T, 3584, 18944)):
    a = torch.randint(-8, 8, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-8, 8, (N, K), dtype=torch.int8, device="cuda")
    ops = 2.0 * M * N * K
    ms = best_ms(lambda: torch._int_mm(a, b.t()))
    print(f"{name} cublas int8: {ops / ms / 1e9:.0f} TOPS ({ms:.3f} ms)", flush=True)
    c = torch.empty((M, N), dtype=torch.int32, device="cuda")
    for bn in ("", "160", "256"):
        if bn:
            os.environ["SPLITQ_TILE_N"] = bn
        else:
            os.environ.pop("SPLITQ_TILE_N", None)
        ms = best_ms(lambda: _lib.check(lib.splitq_gemm_i8(a.data_ptr(), K, 1, b.data_ptr(), K, c.data_ptr(), N,
                                                           M, N, K, None)))
        print(f"{name} splitq raw int8 bn={bn or 'auto'}: {ops / ms / 1e9:.0f} TOPS ({ms:.3f} ms)", flush=True)
    os.environ.pop("SPLITQ_TILE_N", None)
    del a, b, c
    torch.cuda.empty_cache()
    # forward GEMM stage: full layer (aux K) vs no outliers / low-rank (no aux)
    rng = np.random.default_rng(0)
    for k, rs, rc in ((32, wl.default_rank(0.02, K - 64, N), wl.default_rank(0.03, K - 64, N)), (0, 0, 0)):
        spec = wl.LayerSpec(name, K, N, k, k, rs, rc)
        c_t, c_v = wl.outlier_sets(rng, K, max(k, 1))
        c_t, c_v = c_t[:k], c_v[:k]
        layer = wl.build_split_layer(pkg, rng, spec, np.full(K, 4.5), c_t, c_v)
        g = runtime.GpuLayer(layer)
        tags = torch.from_numpy(wl.tags_with_spans(rng, T, T * 5 // 32)).cuda()
        x = torch.randn((T, K), device="cuda").half()
        y = torch.empty((T, N), device="cuda", dtype=torch.float16)
        ws = g.workspace(T)
        for bn in ("", "128", "160") if k else ("", "160"):
            if bn:
                os.environ["SPLITQ_TILE_N"] = bn
            else:
                os.environ.pop("SPLITQ_TILE_N", None)
            for _ in range(2):
                g.run(x, tags, y=y, ws=ws, check=False)
            torch.cuda.synchronize()
            g.profile_read()
            for _ in range(3):
                g.run(x, tags, y=y, ws=ws, check=False, profile=True)
            st, calls = g.profile_read()
            gm = st[2] / calls
            print(f"{name} forward GEMM {'aux k_lr=' + str(g.layout(T).k_lr) if k else 'no aux'} bn={bn or 'auto'}: "
                  f"{ops / gm / 1e9:.0f} TOPS ({gm:.3f} ms)", flush=True)
        os.environ.pop("SPLITQ_TILE_N", None)
        del g, x, y, ws
        torch.cuda.empty_cache()
