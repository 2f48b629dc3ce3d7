"""Split-linear layer mirror (reference: pkg/src/modquant/layer.py).

``forward(layer, batch)`` is the drop-in for layer.py:175-177: it packs the
layer once (weight codes, host fp64, reference operation order), then runs
the whole forward on the GPU through the C-ABI (K1 quantizer -> low-rank
first stages -> tcgen05 split GEMM with fused outliers / low-rank second
stage / merge epilogue). Any object with the reference SplitLayer fields is
accepted, so a ``modquant.layer.SplitLayer`` drops in unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import lowrank
from . import transform as tr
from .mocd import ChannelPartition, trivial_partition
from .quantizer import Granularity, QuantSpec
from .tensor import ActivationBatch, _is_torch, as_matrix

AUX_BITS_FLOOR = 4  # layer.py:38

DEFAULT_ACT_SPEC = QuantSpec(bits=8, symmetric=False, granularity=Granularity.PER_TOKEN)
DEFAULT_WEIGHT_SPEC = QuantSpec(bits=8, symmetric=True, granularity=Granularity.PER_CHANNEL)


@dataclass(frozen=True)
class SplitLayer:  # layer.py:46-97
    partition: ChannelPartition
    w_main: np.ndarray
    w_text: np.ndarray
    w_vision: np.ndarray
    p_main: tr.Transform
    p_text: tr.Transform
    p_vision: tr.Transform
    act_spec: QuantSpec
    weight_spec: QuantSpec
    branch_smooth: lowrank.LowRankBranch | None = None
    branch_comp: lowrank.LowRankBranch | None = None
    use_cws: bool = False
    use_mac: bool = False
    aux_bits_floor: int = AUX_BITS_FLOOR

    def __post_init__(self):
        p = self.partition
        d_out = self.w_main.shape[1]
        if self.w_main.shape[0] != len(p.c_main):
            raise ValueError("w_main rows must match main channel count")
        if self.w_text.shape != (len(p.c_text), d_out):
            raise ValueError("w_text shape mismatch")
        if self.w_vision.shape != (len(p.c_vision), d_out):
            raise ValueError("w_vision shape mismatch")
        for t, width in ((self.p_main, len(p.c_main)), (self.p_text, len(p.c_text)),
                         (self.p_vision, len(p.c_vision))):
            if t.dim != width:
                raise ValueError("transform dim does not match path width")
        if self.use_cws and self.branch_smooth is None:
            raise ValueError("CWS enabled but smoothing branch absent")
        if self.use_mac and self.branch_comp is None:
            raise ValueError("MAC enabled but compensation branch absent")
        for br in (self.branch_smooth, self.branch_comp):
            if br is not None and br.rank > min(len(p.c_main), d_out):
                raise ValueError("branch rank exceeds min(path width, d_out)")

    @property
    def d_out(self) -> int:
        return self.w_main.shape[1]

    def full_weight(self) -> np.ndarray:
        w = np.empty((self.partition.dim, self.d_out))
        w[self.partition.c_main] = self.w_main
        w[self.partition.c_text] = self.w_text
        w[self.partition.c_vision] = self.w_vision
        return w


def build_layer(w, batch, partition=None, act_spec: QuantSpec = DEFAULT_ACT_SPEC,
                weight_spec: QuantSpec = DEFAULT_WEIGHT_SPEC, use_cws: bool = False,
                use_mac: bool = False, rank_ratio_cws: float = 0.02,
                rank_ratio_mac: float = 0.03, smoothing_init: bool = True,
                col_max=None) -> SplitLayer:
    """layer.py:185-232. Offline layer assembly (host): split weights, init the
    diagonal transforms from the calibration activations' column max |X|, and
    anchor the low-rank branches on the SVD of the main weight.

    ``col_max`` (optional) is the per-channel max |X| over the calibration
    tokens, e.g. from the GPU MOCD statistics (``mocd_gpu.channel_absmax``);
    without it the host batch is reduced here, as in transform.py:89.
    """
    w = as_matrix(w)
    if partition is None:
        partition = trivial_partition(w.shape[0])
    if w.shape[0] != partition.dim:
        raise ValueError("weight rows must match partition dim")
    if col_max is None:
        data = np.asarray(batch.data.detach().cpu().double() if _is_torch(batch.data)
                          else batch.data, dtype=np.float64)
        col_max = np.max(np.abs(data), axis=0)
    col_max = np.asarray(col_max, np.float64)

    def _init(idx):
        if not smoothing_init:
            return tr.init_transform(len(idx), "diagonal", None)
        return tr.init_transform(len(idx), "diagonal", col_max[idx])

    p_main = _init(partition.c_main)
    p_text = _init(partition.c_text)
    p_vision = _init(partition.c_vision)
    w_m = w[partition.c_main]
    d_out = w.shape[1]
    branch_smooth = branch_comp = None
    if use_cws:
        r = lowrank.default_rank(rank_ratio_cws, len(partition.c_main), d_out)
        branch_smooth = lowrank.build_branch(w_m, p_main, r)
    if use_mac:
        r = lowrank.default_rank(rank_ratio_mac, len(partition.c_main), d_out)
        branch_comp = lowrank.build_branch(w_m, p_main, r)
    return SplitLayer(
        partition=partition, w_main=w_m, w_text=w[partition.c_text],
        w_vision=w[partition.c_vision], p_main=p_main, p_text=p_text, p_vision=p_vision,
        act_spec=act_spec, weight_spec=weight_spec, branch_smooth=branch_smooth,
        branch_comp=branch_comp, use_cws=use_cws, use_mac=use_mac,
    )


def forward(layer, batch, *, out_dtype=None):
    """y = forward(layer, batch) on the GPU (layer.py:175-177).

    numpy batch -> float64 numpy result (the reference's return type, values
    computed in fp32 on the device); torch CUDA batch -> torch tensor of
    ``out_dtype`` (default float32) left on the device.
    """
    from . import runtime

    return runtime.forward(layer, batch, out_dtype=out_dtype)


def forward_reference(w, batch):
    """Unquantized X @ W (layer.py:180-182) in fp64 on the GPU."""
    import torch

    from . import runtime

    dev = runtime.device()
    x = batch.data
    xt = x.to(dev, torch.float64) if _is_torch(x) else torch.from_numpy(np.asarray(x, np.float64)).to(dev)
    wt = torch.from_numpy(as_matrix(w)).to(dev)
    if xt.shape[1] != wt.shape[0]:
        raise ValueError(f"dimension mismatch: {tuple(xt.shape)} @ {tuple(wt.shape)}")
    y = xt @ wt
    return y if _is_torch(x) else y.cpu().numpy()


def forward_with_cache(layer, batch):
    """layer.py:118-172 on the device: (y fp64 CUDA tensor, cache of fp64 CUDA
    tensors) -- the calibration caller's forward (calib_gpu.py)."""
    from . import calib_gpu

    return calib_gpu.forward_with_cache(layer, batch)


def with_updated_params(layer, p_main=None, p_text=None, p_vision=None, gate_smooth=None,
                        gate_comp=None):
    """layer.py:355-375: a copy with selected learnable parameters replaced."""
    changes = {}
    if p_main is not None:
        changes["p_main"] = p_main
    if p_text is not None:
        changes["p_text"] = p_text
    if p_vision is not None:
        changes["p_vision"] = p_vision
    if gate_smooth is not None:
        changes["branch_smooth"] = layer.branch_smooth.with_gate(gate_smooth)
    if gate_comp is not None:
        changes["branch_comp"] = layer.branch_comp.with_gate(gate_comp)
    return replace(layer, **changes)
