"""B200-native (sm_100a) SplitQ split-linear hot path.

Drop-in for the hot-path subset of the reference package ``modquant``
(pkg/src/modquant/__init__.py): same names and semantics, with the forward,
the per-token activation quantizer and the MOCD calibration statistics
running as hand-written CUDA kernels behind the C-ABI in include/splitq.h.
"""

from .layer import (
    AUX_BITS_FLOOR,
    DEFAULT_ACT_SPEC,
    DEFAULT_WEIGHT_SPEC,
    SplitLayer,
    build_layer,
    forward,
    forward_reference,
    forward_with_cache,
    with_updated_params,
)
from .layer_io import (
    TensorFormatError,
    load_layer,
    load_layer_packed,
    load_packed,
    load_tensor,
    save_layer,
    save_packed,
    save_tensor,
)
from .lowrank import LowRankBranch, SvdFactors, build_branch, default_rank, truncated_svd
from .mocd import ChannelPartition, MocdConfig, jaccard, outlier_set, select_topk, trivial_partition
from .mocd_gpu import build_partition, channel_absmax, percentile_rank, text_score, vision_score
from .calibrate import stability_report
# after the submodule import: ``calibrate`` names the function, as in modquant
from .calib_gpu import CalibConfig, LossTrace, NonFiniteLossError, calibrate
from .quantizer import (
    Granularity,
    QuantParams,
    QuantSpec,
    compute_params,
    fake_quantize,
    quantize,
    quantize_per_token,
)
from .tensor import ActivationBatch, ModalityTag
from .transform import Transform, diagonal_transform, identity_transform, init_transform

__all__ = [
    "AUX_BITS_FLOOR", "DEFAULT_ACT_SPEC", "DEFAULT_WEIGHT_SPEC", "SplitLayer", "build_layer",
    "forward", "forward_reference", "LowRankBranch", "SvdFactors", "build_branch",
    "default_rank", "truncated_svd", "ChannelPartition", "MocdConfig", "select_topk",
    "build_partition", "vision_score", "percentile_rank", "text_score", "channel_absmax", "jaccard",
    "stability_report", "TensorFormatError", "forward_with_cache", "with_updated_params", "CalibConfig",
    "LossTrace", "NonFiniteLossError", "calibrate", "load_tensor", "save_tensor", "load_layer", "save_layer",
    "trivial_partition", "Granularity", "QuantParams", "QuantSpec", "compute_params",
    "fake_quantize", "quantize", "quantize_per_token", "ActivationBatch", "ModalityTag",
    "Transform", "diagonal_transform", "identity_transform", "init_transform",
]
