"""MOCD selection tooling on the device (reference:
pkg/src/modquant/calibrate.py:273-329).

``stability_report`` mirrors the reference: the same stratified token
subsets (the same numpy generator streams, so the same rows), each
partition built by the GPU MOCD statistics (mocd_gpu.build_partition,
bit-identical to the reference's build_partition), and the Jaccard
similarity of the outlier selections to the reference-size selection.
The subsets are gathered on the device; a CUDA batch never leaves it.
"""

from __future__ import annotations

import numpy as np

from . import mocd_gpu
from .mocd import MocdConfig, jaccard, outlier_set
from .tensor import _is_torch


def _rows_of(tags, value):
    return np.flatnonzero(np.asarray(tags) == value).astype(np.int64)


def _stratified_subset(rng, tags, size: int) -> np.ndarray:  # calibrate.py:273-290
    """Token subset keeping roughly the batch's text/vision proportions."""
    t_rows, v_rows = _rows_of(tags, 0), _rows_of(tags, 1)
    total = int(np.asarray(tags).shape[0])
    if size > total:
        raise ValueError(f"subset size {size} exceeds {total} tokens")
    n_t = int(round(size * t_rows.size / total))
    if t_rows.size:
        n_t = min(max(n_t, 1), t_rows.size, size)
    n_v = size - n_t
    if v_rows.size and n_v == 0 and size > 1:
        n_v, n_t = 1, size - 1
    chosen = np.concatenate([
        rng.choice(t_rows, size=n_t, replace=False) if n_t else np.empty(0, np.int64),
        rng.choice(v_rows, size=n_v, replace=False) if n_v else np.empty(0, np.int64),
    ])
    return np.sort(chosen.astype(np.int64))


def _partition(x, tags_np, rows, cfg):
    """build_partition of the rows' subset, gathered on the device."""
    import torch

    if _is_torch(x):
        idx = torch.from_numpy(rows).to(x.device)
        xs = x.index_select(0, idx)
    else:
        xs = np.asarray(x)[rows]
    return mocd_gpu.build_partition_distributed(xs, tags_np[rows], cfg, group=False)


def stability_report(batch, cfg: MocdConfig, subset_sizes: list[int], reference_size: int,
                     trials: int, seed: int = 0) -> list[dict]:  # calibrate.py:301-329
    """Mean / std Jaccard similarity of outlier selections from random token
    subsets against the reference-size selection."""
    tags = batch.tags.cpu().numpy() if _is_torch(batch.tags) else np.asarray(batch.tags, np.uint8)
    total = int(tags.shape[0])
    if reference_size > total:
        raise ValueError("reference size exceeds token count")
    ref_rng = np.random.default_rng(seed)
    ref_rows = _stratified_subset(ref_rng, tags, reference_size)
    ref_sel = outlier_set(_partition(batch.data, tags, ref_rows, cfg))
    report = []
    for size in subset_sizes:
        sims = []
        for trial in range(trials):
            rng = np.random.default_rng(seed * 1_000_003 + trial + 1)
            rows = _stratified_subset(rng, tags, size)
            sel = outlier_set(_partition(batch.data, tags, rows, cfg))
            sims.append(jaccard(sel, ref_sel))
        sims = np.asarray(sims)
        report.append({"subset_size": size, "mean_jaccard": float(sims.mean()),
                       "std_jaccard": float(sims.std())})
    return report
