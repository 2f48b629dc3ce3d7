"""Activation batch mirror (reference: pkg/src/modquant/tensor.py:27-80).

``ActivationBatch`` accepts numpy arrays (validated like the reference, kept
as float64) or torch tensors (kept on their device; a CUDA batch never
round-trips through the host).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np


class ModalityTag(enum.IntEnum):  # tensor.py:27-29
    TEXT = 0
    VISION = 1


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def as_matrix(values, rows=None, cols=None):
    """tensor.py:32-47 (numpy inputs)."""
    m = np.asarray(values, dtype=np.float64)
    if m.ndim != 2:
        raise ValueError(f"matrix must be 2-D, got ndim={m.ndim}")
    if not np.all(np.isfinite(m)):
        raise ValueError("non-finite value in matrix")
    if rows is not None and m.shape[0] != rows:
        raise ValueError(f"expected {rows} rows, got {m.shape[0]}")
    if cols is not None and m.shape[1] != cols:
        raise ValueError(f"expected {cols} cols, got {m.shape[1]}")
    return np.ascontiguousarray(m)


@dataclass(frozen=True)
class ActivationBatch:  # tensor.py:50-80
    data: object
    tags: object

    def __post_init__(self):
        if _is_torch(self.data):
            if self.data.ndim != 2:
                raise ValueError(f"matrix must be 2-D, got ndim={self.data.ndim}")
            n = self.data.shape[0]
            tags = self.tags
            if not _is_torch(tags):
                import torch
                tags = torch.as_tensor(np.asarray(tags, dtype=np.uint8), device=self.data.device)
            tags = tags.to(dtype=__import__("torch").uint8)
            if tags.ndim != 1:
                raise ValueError("tags must be a 1-D sequence")
            if tags.shape[0] != n:
                raise ValueError("tag-length mismatch")
            if n < 1:
                raise ValueError("batch must contain at least one token")
            object.__setattr__(self, "tags", tags)
            return
        object.__setattr__(self, "data", as_matrix(self.data))
        tags = np.asarray(self.tags, dtype=np.uint8)
        if tags.ndim != 1:
            raise ValueError("tags must be a 1-D sequence")
        if tags.shape[0] != self.data.shape[0]:
            raise ValueError("tag-length mismatch")
        if self.data.shape[0] < 1:
            raise ValueError("batch must contain at least one token")
        if not np.all((tags == ModalityTag.TEXT) | (tags == ModalityTag.VISION)):
            raise ValueError("tags must be 0 (text) or 1 (vision)")
        object.__setattr__(self, "tags", tags)

    @property
    def text_rows(self):
        t = self.tags
        if _is_torch(t):
            return (t == 0).nonzero().flatten()
        return np.flatnonzero(t == ModalityTag.TEXT)

    @property
    def vision_rows(self):
        t = self.tags
        if _is_torch(t):
            return (t == 1).nonzero().flatten()
        return np.flatnonzero(t == ModalityTag.VISION)
