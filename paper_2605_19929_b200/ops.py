"""PyTorch custom ops over the C-ABI (north star: "Python host code and PyTorch
custom ops call a thin C-ABI layer").

``torch.ops.splitq.forward`` and ``torch.ops.splitq.quantize_per_token`` are
registered with ``torch.library.custom_op``: opaque to autograd / dynamo, with
fake (meta) implementations so ``torch.compile`` and FakeTensor tracing see
their output shapes, and no host synchronisation on the launch path, so both
can be captured in a CUDA graph. The device work is the same libsplitq_b200.so
call as ``GpuLayer.run`` / ``quantize_rows``; status words are read by
``check_status`` when the caller chooses (the reference raises ValueError on
non-finite inputs: tensor.py:39-40).

A packed layer is referenced by an integer id (``register_layer``), since
custom-op schemas take tensors and scalars only.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .runtime import GpuLayer, _dtype_code, _ptr, _spec_struct, _stream, packed

_LAYERS: dict[int, GpuLayer] = {}
_OUT_DTYPES = {0: torch.float32, 1: torch.float16, 2: torch.bfloat16}
_OUT_CODES = {v: k for k, v in _OUT_DTYPES.items()}


def register_layer(layer) -> int:
    """Pack a SplitLayer (or take a GpuLayer) and return the id the ops take."""
    g = packed(layer)
    key = id(g)
    _LAYERS[key] = g
    return key


def _layer(layer_id: int) -> GpuLayer:
    g = _LAYERS.get(int(layer_id))
    if g is None:
        raise ValueError(f"unknown splitq layer id {layer_id} (use register_layer)")
    return g


@torch.library.custom_op("splitq::forward", mutates_args=("ws",))
def forward_op(x: torch.Tensor, tags: torch.Tensor, ws: torch.Tensor, layer_id: int,
               out_code: int) -> torch.Tensor:
    """y = forward(layer, batch) (layer.py:175-177): fp32 / fp16 / bf16
    [T x d_out]; ``ws`` is the caller-owned workspace (``workspace_for``) whose
    first int32 is the status word."""
    g = _layer(layer_id)
    return g.run(x, tags, out_dtype=_OUT_DTYPES[int(out_code)], ws=ws, check=False)


@forward_op.register_fake
def _(x, tags, ws, layer_id, out_code):
    g = _layer(layer_id)
    return x.new_empty((x.shape[0], g.d_out), dtype=_OUT_DTYPES[int(out_code)])


@torch.library.custom_op("splitq::quantize_per_token", mutates_args=())
def quantize_per_token_op(x: torch.Tensor, bits: int, symmetric: bool
                          ) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    """PER_TOKEN compute_params + codes (quantizer.py:104-155) on the device:
    (codes int8 [rows x roundup(cols, 16)], scales f64 [rows], zero points
    i32 [rows], status i32 [4]). Codes are stored centred (q - zp, int8) when
    ``symmetric or bits <= 7``, else as u8 q (viewed as int8)."""
    lib = _lib.load()
    if x.ndim != 2:
        raise ValueError(f"matrix must be 2-D, got ndim={x.ndim}")
    if x.stride(1) != 1:
        x = x.contiguous()
    rows, cols = int(x.shape[0]), int(x.shape[1])
    ld = (cols + 15) // 16 * 16
    codes = torch.empty((rows, ld), dtype=torch.int8, device=x.device)
    scales = torch.empty(rows, dtype=torch.float64, device=x.device)
    zps = torch.empty(rows, dtype=torch.int32, device=x.device)
    status = torch.zeros(4, dtype=torch.int32, device=x.device)
    if rows and cols:
        from .quantizer import Granularity, QuantSpec

        spec = _spec_struct(QuantSpec(int(bits), bool(symmetric), Granularity.PER_TOKEN))
        centered = C.c_int32()
        _lib.check(lib.splitq_quantize_rows(_ptr(x), _dtype_code(x.dtype), x.stride(0), rows, cols, spec,
                                            _ptr(codes), ld, _ptr(scales), _ptr(zps), _ptr(status),
                                            C.byref(centered), _stream()))
    return codes, scales, zps, status


@quantize_per_token_op.register_fake
def _(x, bits, symmetric):
    rows, cols = x.shape
    ld = (cols + 15) // 16 * 16
    return (x.new_empty((rows, ld), dtype=torch.int8), x.new_empty((rows,), dtype=torch.float64),
            x.new_empty((rows,), dtype=torch.int32), x.new_empty((4,), dtype=torch.int32))


def workspace_for(layer_id: int, tokens: int) -> torch.Tensor:
    """A fresh workspace for ``tokens`` rows of the layer (caller-owned)."""
    g = _layer(layer_id)
    return torch.empty(int(g.layout(tokens).total_bytes), dtype=torch.uint8, device=g.device)


def check_status(status: torch.Tensor) -> None:
    """Raise the reference's ValueError for a non-zero status word (the first
    int32 of a forward workspace, or the quantize op's status tensor)."""
    _lib.check(_lib.load().splitq_read_status(_ptr(status), _stream(), C.byref(C.c_int32())))


def forward(layer_id: int, x: torch.Tensor, tags: torch.Tensor, ws: torch.Tensor,
            out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    return torch.ops.splitq.forward(x, tags, ws, layer_id, _OUT_CODES[out_dtype])
