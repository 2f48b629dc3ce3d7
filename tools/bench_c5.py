#!/usr/bin/env python
"""BASELINE config 5: the MOCD calibration-statistics pass and the 28-layer
W4A4 forward over the same 128 x 2048 synthetic tokens (25 % vision), on
1..8 GPUs of one node.

Single GPU:  python tools/bench_c5.py
N GPUs:      python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
                 --master-addr 127.0.0.1 --master-port P tools/bench_c5.py

The 128 samples are sharded across the ranks (token rows). MOCD
(mocd.py:153-179, mocd_gpu.build_partition_distributed): every rank reduces
its own rows; the per-channel absmax is MAX-all-reduced over NCCL, the rank
counts (percentile_rank numerators) go through one all-to-all so that each
rank holds every text row of its own channel range, the k-means text scores
are SUM-all-reduced, and the top-k runs identically on every rank. Per layer
input width (3584 for the q/k/v, o and gate/up inputs; 18944 for the down
input) one build_partition; times are CUDA-synchronised wall clock, max over
ranks. The 28-layer forward applies 28 x 7 split-linear projections to the
rank's tokens (no collective: rows are independent); the 28 layers reuse 7
packed weight sets (each layer's weights still stream from HBM: the 7 sets
are 1.7 GB, far above L2). Rank 0 prints one JSON line.
"""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import workloads as wl  # noqa: E402
import paper_2605_19929_b200 as pkg  # noqa: E402
from paper_2605_19929_b200 import mocd_gpu, runtime  # noqa: E402

SAMPLES, SEQ = 128, 2048
world, rank, local = bench.dist_env()
if world > 1:
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
dev = torch.device("cuda", torch.cuda.current_device())
if SAMPLES % world:
    raise SystemExit(f"{SAMPLES} samples do not split over {world} ranks")
my_samples = SAMPLES // world
T = my_samples * SEQ
tags = np.concatenate([wl.tags_with_spans(np.random.default_rng((5, s)), SEQ, SEQ // 4)
                       for s in range(rank * my_samples, (rank + 1) * my_samples)])
tg = torch.from_numpy(tags).to(dev)
peaks = bench.measured_peaks()
hbm = peaks.get("hbm_gbs", 6535.4)
out = {"config": "config5: 128 x 2048 tokens (25% vision); MOCD statistics per layer-input width + "
                 "28-layer Qwen2.5-VL-7B W4A4 forward", "tokens": SAMPLES * SEQ, "n_gpus": world,
       "tokens_per_gpu": T, "hbm_peak_gbs": hbm,
       "parallelism": f"dp{world}: samples sharded; MOCD MAX all-reduce + all-to-all + SUM all-reduce "
                      "(NCCL when N > 1)"}


def sync():
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()


def max_over_ranks(v):
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed(fn, reps=3):
    fn()
    best = 1e9
    r = None
    for _ in range(reps):
        sync()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return max_over_ranks(best), r


mocd = {}
for d_in in (3584, 18944):
    prng = np.random.default_rng((7, d_in))  # the planted sets: identical on every rank
    spec_in = {"d_in": d_in, "c_t": np.sort(prng.permutation(d_in)[:32]),
               "c_v": np.sort(prng.permutation(d_in)[32:64]),
               "scales_t": prng.uniform(30, 100, 32), "scales_v": prng.uniform(30, 100, 32)}
    x = bench.make_input_tensor(torch, dev, T, spec_in, tags, 11 + rank)
    cfg = pkg.MocdConfig(0.01, 0.01)
    st = mocd_gpu._GPU
    t_abs, (vmax, amax) = timed(lambda: st.absmax(x, tg))
    t_part, part = timed(lambda: mocd_gpu.build_partition_distributed(x, tg, cfg), reps=1)
    abs_bytes = T * d_in * 2
    mocd[str(d_in)] = {
        "absmax_ms": t_abs * 1e3, "absmax_gbs_per_gpu": abs_bytes / t_abs / 1e9,
        "absmax_frac_hbm": abs_bytes / t_abs / 1e9 / hbm,
        "build_partition_ms": t_part * 1e3,
        "partition_sizes": [len(part.c_main), len(part.c_text), len(part.c_vision)],
    }
    if world == 1:  # stage split of the single-GPU pass
        cand = np.setdiff1d(np.arange(d_in), np.asarray(st.topk(vmax, cfg.k_vision(d_in)).cpu()))
        t_rank, counts = timed(lambda: st.rank_counts(x, tg, cand), reps=1)
        n_text = int(counts.shape[0])
        t_score, _ = timed(lambda: st.text_score(counts, cand.size, min(cfg.clusters_k, n_text),
                                                 cfg.kmeans_max_iter), reps=1)
        mocd[str(d_in)].update(rank_counts_ms=t_rank * 1e3, text_rows=n_text, candidates=int(cand.size),
                               text_score_ms=t_score * 1e3)
        del counts
    del x
    torch.cuda.empty_cache()
out["mocd"] = mocd
# 28 x (3 MOCD passes at 3584 + 1 at 18944): the whole calibration-statistics job
out["mocd_28_layers_s"] = 28 * (3 * mocd["3584"]["build_partition_ms"] +
                                mocd["18944"]["build_partition_ms"]) / 1e3

# ---------------------------------------------------------------- 28-layer forward
tags_w, inputs, layers = bench.build_workload(pkg, SEQ, 4, 4)
gls = [(g, sp, runtime.GpuLayer(layer, dev)) for g, sp, layer in layers]
xs = {g: bench.make_input_tensor(torch, dev, T, inputs[g], tags, 20 + 97 * rank + i) for i, g in enumerate(inputs)}
ws = torch.empty(max(int(gl.layout(T).total_bytes) for _, _, gl in gls), dtype=torch.uint8, device=dev)
ys = {sp.name: torch.empty((T, sp.d_out), dtype=torch.float16, device=dev) for _, sp, _ in gls}


def forward28():
    for _ in range(28):
        for g, sp, gl in gls:
            gl.run(xs[g], tg, y=ys[sp.name], check=False, ws=ws)


forward28()
sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
forward28()
e1.record()
e1.synchronize()
ms = max_over_ranks(e0.elapsed_time(e1))
ops = 28 * SAMPLES * SEQ * sum(2 * sp.d_in * sp.d_out for _, sp, _ in gls)
out["forward_28_layers_ms"] = ms
out["forward_28_layers_tokens_per_s"] = SAMPLES * SEQ / (ms * 1e-3)
out["forward_28_layers_tops_dense_equiv"] = ops / (ms * 1e-3) / 1e12
if rank == 0:
    print(json.dumps(out), flush=True)
if world > 1:
    dist.destroy_process_group()
