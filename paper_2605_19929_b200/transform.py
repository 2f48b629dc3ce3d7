"""Diagonal per-path transform mirror (reference: pkg/src/modquant/transform.py).

Only the diagonal family is on the split-linear path (build_layer creates
diagonal transforms, layer.py:209-211). ``Transform.scale`` evaluates
exp(log_scale) exactly like the reference (transform.py:37-39); the GPU
consumes that fp64 vector and never recomputes exp/log on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DIAG_EPS = 1e-6
DIAG_MAX = 1e6
SMOOTHING_ALPHA = 0.5


@dataclass(frozen=True)
class Transform:  # transform.py:24-39 (diagonal members)
    dim: int
    log_scale: np.ndarray | None = None
    dense: np.ndarray | None = None

    @property
    def is_diagonal(self) -> bool:
        return self.log_scale is not None

    @property
    def scale(self) -> np.ndarray:
        return np.exp(self.log_scale)


def diagonal_transform(scale) -> Transform:  # transform.py:42-51
    scale = np.asarray(scale, dtype=np.float64)
    if scale.ndim != 1:
        raise ValueError("diagonal scale must be 1-D")
    mag = np.abs(scale)
    if np.any(mag < DIAG_EPS) or np.any(mag > DIAG_MAX):
        raise ValueError(f"diagonal magnitudes must lie in [{DIAG_EPS}, {DIAG_MAX}]")
    if np.any(scale <= 0):
        raise ValueError("diagonal scales must be positive (log parameterization)")
    return Transform(dim=scale.shape[0], log_scale=np.log(scale))


def identity_transform(dim: int) -> Transform:
    return diagonal_transform(np.ones(dim)) if dim > 0 else Transform(0, np.zeros(0))


def smoothing_scale_from_colmax(col_max) -> np.ndarray:
    """d = clip(max(col_max, eps) ** alpha, eps, max) (transform.py:89-91);
    col_max is the per-channel max |X| (the MOCD absmax statistic)."""
    col_max = np.asarray(col_max, dtype=np.float64)
    return np.clip(np.maximum(col_max, DIAG_EPS) ** SMOOTHING_ALPHA, DIAG_EPS, DIAG_MAX)


def init_transform(dim: int, kind: str = "diagonal", x_calib=None) -> Transform:
    """transform.py:75-91 (diagonal kind). ``x_calib`` may be a numpy matrix or
    a precomputed per-channel absmax vector (``col_max=``-style 1-D input)."""
    if kind != "diagonal":
        raise ValueError(f"unsupported transform kind {kind!r} on the GPU path")
    if dim == 0:
        return Transform(0, np.zeros(0))
    if x_calib is None or np.size(x_calib) == 0:
        return diagonal_transform(np.ones(dim))
    x_calib = np.asarray(x_calib, dtype=np.float64)
    if x_calib.ndim == 1:
        col_max = x_calib
    else:
        if x_calib.shape[1] != dim:
            raise ValueError(f"expected {dim} cols, got {x_calib.shape[1]}")
        if not np.all(np.isfinite(x_calib)):
            raise ValueError("non-finite value in matrix")
        col_max = np.max(np.abs(x_calib), axis=0)
    return diagonal_transform(smoothing_scale_from_colmax(col_max))
