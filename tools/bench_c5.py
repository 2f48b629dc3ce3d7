#!/usr/bin/env python
"""BASELINE config 5 on one GPU: the MOCD calibration-statistics pass and the
28-layer W4A4 forward over the same 128 x 2048 synthetic tokens (25 % vision).

MOCD (mocd.py:153-179 on the GPU, csrc/mocd.cu): per layer input width
(3584 for the q/k/v, o and gate/up inputs; 18944 for the down input) one
build_partition over the 262,144 calibration tokens, timed per kernel stage:
  absmax  (vision_score + init_transform column max)  -- HBM-bound: 2 B / element
  rank counts (percentile_rank numerators, text rows) -- per-row SMEM rank
  text score (exact 1-D k-means per candidate channel)
The 28-layer forward applies 28 x 7 split-linear projections to the same
tokens; the 28 layers reuse 7 packed weight sets (each layer's weights still
stream from HBM: the 7 sets are 1.7 GB, far above L2).
Prints one JSON line.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import workloads as wl  # noqa: E402
import paper_2605_19929_b200 as pkg  # noqa: E402
from paper_2605_19929_b200 import mocd_gpu, runtime  # noqa: E402

SAMPLES, SEQ = 128, 2048
dev = torch.device("cuda", 0)
T = SAMPLES * SEQ
rng = np.random.default_rng(5)
tags = np.concatenate([wl.tags_with_spans(rng, SEQ, SEQ // 4) for _ in range(SAMPLES)])
tg = torch.from_numpy(tags).to(dev)
peaks = bench.measured_peaks()
hbm = peaks.get("hbm_gbs", 6535.4)
out = {"config": "config5: 128 x 2048 tokens (25% vision); MOCD statistics per layer-input width + "
                 "28-layer Qwen2.5-VL-7B W4A4 forward", "tokens": T, "hbm_peak_gbs": hbm}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best, r


mocd = {}
for d_in in (3584, 18944):
    spec_in = {"d_in": d_in, "c_t": np.sort(rng.permutation(d_in)[:32]),
               "c_v": np.sort(rng.permutation(d_in)[32:64]),
               "scales_t": rng.uniform(30, 100, 32), "scales_v": rng.uniform(30, 100, 32)}
    x = bench.make_input_tensor(torch, dev, T, spec_in, tags, 11)
    cfg = pkg.MocdConfig(0.01, 0.01)
    st = mocd_gpu._GPU
    t_abs, (vmax, amax) = timed(lambda: st.absmax(x, tg))
    cand = np.setdiff1d(np.arange(d_in), np.asarray(st.topk(vmax, cfg.k_vision(d_in)).cpu()))
    t_rank, counts = timed(lambda: st.rank_counts(x, tg, cand), reps=1)
    n_text = int(counts.shape[0])
    t_score, scores = timed(lambda: st.text_score(counts, cand.size, min(cfg.clusters_k, n_text),
                                                  cfg.kmeans_max_iter), reps=1)
    t_part, part = timed(lambda: mocd_gpu.build_partition(pkg.ActivationBatch(x, tg), cfg), reps=1)
    abs_bytes = T * d_in * 2
    mocd[str(d_in)] = {
        "absmax_ms": t_abs * 1e3, "absmax_gbs": abs_bytes / t_abs / 1e9,
        "absmax_frac_hbm": abs_bytes / t_abs / 1e9 / hbm,
        "rank_counts_ms": t_rank * 1e3, "text_rows": n_text, "candidates": int(cand.size),
        "rank_counts_rows_per_s": n_text / t_rank,
        "text_score_ms": t_score * 1e3, "text_score_channels_per_s": cand.size / t_score,
        "build_partition_ms": t_part * 1e3,
        "partition_sizes": [len(part.c_main), len(part.c_text), len(part.c_vision)],
    }
    del x, counts
    torch.cuda.empty_cache()
out["mocd"] = mocd
# 28 x (3 MOCD passes at 3584 + 1 at 18944): the whole calibration-statistics job
out["mocd_28_layers_s"] = 28 * (3 * mocd["3584"]["build_partition_ms"] +
                                mocd["18944"]["build_partition_ms"]) / 1e3

# ---------------------------------------------------------------- 28-layer forward
tags_w, inputs, layers = bench.build_workload(pkg, SEQ, 4, 4)
gls = [(g, sp, runtime.GpuLayer(layer, dev)) for g, sp, layer in layers]
xs = {g: bench.make_input_tensor(torch, dev, T, inputs[g], tags, 20 + i) for i, g in enumerate(inputs)}
ws = torch.empty(max(int(gl.layout(T).total_bytes) for _, _, gl in gls), dtype=torch.uint8, device=dev)
ys = {sp.name: torch.empty((T, sp.d_out), dtype=torch.float16, device=dev) for _, sp, _ in gls}


def forward28():
    for _ in range(28):
        for g, sp, gl in gls:
            gl.run(xs[g], tg, y=ys[sp.name], check=False, ws=ws)


forward28()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
forward28()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1)
ops = 28 * T * sum(2 * sp.d_in * sp.d_out for _, sp, _ in gls)
out["forward_28_layers_ms"] = ms
out["forward_28_layers_tokens_per_s"] = T / (ms * 1e-3)
out["forward_28_layers_tops_dense_equiv"] = ops / (ms * 1e-3) / 1e12
print(json.dumps(out), flush=True)
