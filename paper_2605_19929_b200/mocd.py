"""MOCD channel partition types (reference: pkg/src/modquant/mocd.py:19-69).

The GPU calibration statistics (vision saliency, column absmax, text
response-consistency ranks and k-means scores) live in ``mocd_gpu``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ChannelPartition:  # mocd.py:19-42
    c_main: np.ndarray
    c_text: np.ndarray
    c_vision: np.ndarray
    dim: int

    def __post_init__(self):
        for name in ("c_main", "c_text", "c_vision"):
            arr = np.asarray(getattr(self, name), dtype=np.int64)
            if arr.size and (np.any(np.diff(arr) <= 0)):
                raise ValueError(f"{name} must be strictly ascending")
            object.__setattr__(self, name, arr)
        total = np.concatenate([self.c_main, self.c_text, self.c_vision])
        if len(np.unique(total)) != len(total):
            raise ValueError("channel sets must be pairwise disjoint")
        if len(total) != self.dim or (
            self.dim and (total.min() < 0 or total.max() >= self.dim)
        ):
            raise ValueError("channel sets must cover exactly 0..dim-1")
        if len(self.c_main) < len(self.c_text) or len(self.c_main) < len(self.c_vision):
            raise ValueError("main set must be at least as large as each outlier set")


def trivial_partition(dim: int) -> ChannelPartition:  # mocd.py:45-46
    return ChannelPartition(np.arange(dim), np.empty(0, np.int64), np.empty(0, np.int64), dim)


@dataclass(frozen=True)
class MocdConfig:  # mocd.py:49-69
    ratio_vision: float = 0.02
    ratio_text: float = 0.02
    clusters_k: int = 3
    kmeans_max_iter: int = 50
    seed: int = 0

    def __post_init__(self):
        for name in ("ratio_vision", "ratio_text"):
            r = getattr(self, name)
            if not 0.0 <= r <= 0.5:
                raise ValueError(f"{name} must be in [0, 0.5], got {r}")
        if self.clusters_k < 1:
            raise ValueError("clusters_k must be positive")

    def k_vision(self, dim: int) -> int:
        return int(np.floor(self.ratio_vision * dim + 0.5))

    def k_text(self, dim: int) -> int:
        return int(np.floor(self.ratio_text * dim + 0.5))


def select_topk(scores, k: int) -> np.ndarray:  # mocd.py:80-89
    """Indices of the k largest scores, ties to the lower index, ascending.
    O(D) selection over the final (tiny) score vector."""
    scores = np.asarray(scores, dtype=np.float64)
    if k > scores.shape[0]:
        raise ValueError(f"k={k} exceeds score vector length {scores.shape[0]}")
    if k == 0:
        return np.empty(0, dtype=np.int64)
    order = np.argsort(-scores, kind="stable")
    return np.sort(order[:k]).astype(np.int64)


def jaccard(a, b) -> float:  # mocd.py:182-190
    """|A n B| / |A u B|; two empty sets count as identical (1.0)."""
    sa = set(np.asarray(a, dtype=np.int64).tolist())
    sb = set(np.asarray(b, dtype=np.int64).tolist())
    union = sa | sb
    return 1.0 if not union else len(sa & sb) / len(union)


def outlier_set(partition) -> np.ndarray:  # calibrate.py:297-298
    return np.sort(np.concatenate([partition.c_text, partition.c_vision]))
