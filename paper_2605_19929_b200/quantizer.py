"""Quantizer API mirror (reference: pkg/src/modquant/quantizer.py).

``QuantSpec`` / ``Granularity`` / ``QuantParams`` keep the reference's names,
fields and validation messages (quantizer.py:21-73). Activation quantization
(PER_TOKEN) runs on the GPU through the C-ABI (``splitq_quantize_rows``,
K1 in csrc/quantize.cuh). Weight quantization is offline layer packing and
uses the host fp64 expressions below, in the reference's operation order, so
the packed weight codes are identical to the reference's by construction.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, replace

import numpy as np


class Granularity(enum.Enum):  # quantizer.py:21-24
    PER_TENSOR = "per_tensor"
    PER_CHANNEL = "per_channel"  # one group per column
    PER_TOKEN = "per_token"      # one group per row


@dataclass(frozen=True)
class QuantSpec:  # quantizer.py:27-57
    bits: int | None
    symmetric: bool
    granularity: Granularity

    def __post_init__(self):
        if self.bits is not None and not 2 <= self.bits <= 16:
            raise ValueError(f"bits must be in [2, 16] or None, got {self.bits}")

    @property
    def is_identity(self) -> bool:
        return self.bits is None

    @property
    def q_min(self) -> int:
        if self.symmetric:
            return -(2 ** (self.bits - 1)) + 1
        return 0

    @property
    def q_max(self) -> int:
        if self.symmetric:
            return 2 ** (self.bits - 1) - 1
        return 2 ** self.bits - 1

    def with_floor(self, min_bits: int) -> "QuantSpec":
        if self.bits is None or self.bits >= min_bits:
            return self
        return replace(self, bits=min_bits)


@dataclass(frozen=True)
class QuantParams:  # quantizer.py:60-73
    scales: np.ndarray
    zero_points: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "scales", np.asarray(self.scales, dtype=np.float64))
        object.__setattr__(self, "zero_points", np.asarray(self.zero_points, dtype=np.int64))
        if np.any(self.scales <= 0):
            raise ValueError("scales must be positive")


def gpu_spec_supported(spec) -> bool:
    """The integer GPU path covers bits 2..8 (int8 tensor-core operands)."""
    return spec.bits is not None and 2 <= spec.bits <= 8


# ---------------------------------------------------------------- host weight side

def _round_half_away(x):
    return np.sign(x) * np.floor(np.abs(x) + 0.5)  # quantizer.py:76-77


def weight_codes(m: np.ndarray, spec) -> tuple[np.ndarray, np.ndarray]:
    """Centred integer codes (q - z) and per-column fp64 scales of
    fake_quantize(m, compute_params(m, spec), spec) for a weight matrix
    (quantizer.py:104-155 with PER_CHANNEL / PER_TENSOR groups)."""
    m = np.asarray(m, dtype=np.float64)
    gran = spec.granularity.value if hasattr(spec.granularity, "value") else spec.granularity
    if gran == "per_token":
        raise ValueError("weight quantization must be per_channel or per_tensor on the GPU path")
    if not np.all(np.isfinite(m)):
        raise ValueError("non-finite value in matrix")
    q_min, q_max = spec.q_min, spec.q_max
    n = m.shape[1]
    if m.size == 0:
        return np.zeros(m.shape, np.int64), np.ones(n)
    axis = 0 if gran == "per_channel" else None
    if spec.symmetric:
        absmax = np.atleast_1d(np.max(np.abs(m), axis=axis))
        scales = np.where(absmax > 0, absmax / q_max, 1.0)
        zps = np.zeros_like(scales, dtype=np.int64)
    else:
        lo = np.atleast_1d(np.min(m, axis=axis))
        hi = np.atleast_1d(np.max(m, axis=axis))
        span = hi - lo
        const = span == 0
        lo = np.where(const, np.minimum(lo, 0.0), lo)
        hi = np.where(const, np.maximum(hi, 0.0), hi)
        span = hi - lo
        scales = np.where(span > 0, span / (q_max - q_min), 1.0)
        zps = np.clip(_round_half_away(-lo / scales), q_min, q_max).astype(np.int64)
    if np.any(scales <= 0):
        raise ValueError("scales must be positive")
    s = scales.reshape(1, -1)
    z = zps.astype(np.float64).reshape(1, -1)
    q = np.clip(_round_half_away(m / s) + z, q_min, q_max)
    qc = (q - z).astype(np.int64)
    if scales.shape[0] == 1 and n != 1:
        scales = np.full(n, scales[0])
    return qc, scales


# ---------------------------------------------------------------- GPU activation side

def quantize_per_token(x, spec: QuantSpec):
    """PER_TOKEN compute_params + codes on the GPU (K1 kernel).

    ``x``: torch CUDA tensor or array-like [rows x cols] (f16/bf16/f32/f64).
    Returns (codes int64 ndarray of q, QuantParams) exactly as the reference's
    compute_params / fake_quantize define them (quantizer.py:104-155).
    """
    from . import runtime

    return runtime.quantize_rows(x, spec)


def compute_params(m, spec: QuantSpec) -> QuantParams:
    """GPU compute_params for PER_TOKEN specs (the activation hot path)."""
    _check_token_spec(spec)
    _, params = quantize_per_token(m, spec)
    return params


def fake_quantize(m, params: QuantParams, spec: QuantSpec):
    """(q - z) * S for PER_TOKEN specs; params must come from the same data
    (they are recomputed on the GPU and checked)."""
    _check_token_spec(spec)
    q, p = quantize_per_token(m, spec)
    if params.scales.shape != p.scales.shape or not np.array_equal(params.scales, p.scales) \
            or not np.array_equal(params.zero_points, p.zero_points):
        raise ValueError("fake_quantize on the GPU path requires the params of the same data")
    return (q - p.zero_points[:, None]).astype(np.float64) * p.scales[:, None]


def quantize(m, spec: QuantSpec):
    """quantize() (quantizer.py:170-172) for PER_TOKEN specs on the GPU."""
    _check_token_spec(spec)
    q, p = quantize_per_token(m, spec)
    return (q - p.zero_points[:, None]).astype(np.float64) * p.scales[:, None]


def _check_token_spec(spec):
    if spec.granularity is not Granularity.PER_TOKEN and getattr(
            spec.granularity, "value", spec.granularity) != "per_token":
        raise ValueError("the GPU quantizer implements PER_TOKEN (activation) granularity")
    if not gpu_spec_supported(spec):
        raise ValueError(f"GPU quantizer supports bits 2..8, got {spec.bits}")
