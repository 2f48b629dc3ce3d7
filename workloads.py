"""Seeded synthetic workloads for the BASELINE.json configs (bench / tests).

No public dataset or checkpoint is involved: activations and weights are
drawn from fixed-seed numpy generators with the shapes, modality mixes and
outlier distributions BASELINE.json states.

  C1  single layer 2048->2048, 512 tokens (384 vision then 128 text), W4A4,
      x50 outliers on channels 0-15 (text rows) / 16-31 (vision rows),
      explicit partition C_t = 0..15, C_v = 16..31, CWS + MAC rank 16 with
      factors N(0, 0.01).
  C2  Qwen2.5-VL-3B projections (hidden 2048, inter 11008, kv 256).
  C3  Qwen2.5-VL-7B projections (hidden 3584, inter 18944, kv 512),
      8192-token samples (1280 vision in contiguous spans + 6912 text).
  C4  7B shapes at W3A3 / W3A2 (prefill and decode).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

QWEN_7B = dict(hidden=3584, inter=18944, kv=512, k_out=32)
QWEN_3B = dict(hidden=2048, inter=11008, kv=256, k_out=None)  # K = round(1% of D_in)


def projections(shape: dict):
    h, i, kv = shape["hidden"], shape["inter"], shape["kv"]
    return [("q", h, h), ("k", h, kv), ("v", h, kv), ("o", h, h),
            ("gate", h, i), ("up", h, i), ("down", i, h)]


def default_rank(ratio, path_width, d_out):  # lowrank.py:88-93
    full = min(path_width, d_out)
    return 0 if full == 0 else max(1, int(np.floor(ratio * full + 0.5)))


@dataclass
class LayerSpec:
    name: str
    d_in: int
    d_out: int
    k_text: int
    k_vision: int
    r_cws: int
    r_mac: int
    abits: int = 4
    wbits: int = 4
    a_sym: bool = False


def tags_with_spans(rng, tokens, n_vision):
    """Vision tokens as a few contiguous image spans inside a text sequence."""
    tags = np.zeros(tokens, np.uint8)
    if n_vision == 0:
        return tags
    n_spans = max(1, min(4, n_vision // 256))
    sizes = np.full(n_spans, n_vision // n_spans)
    sizes[: n_vision - sizes.sum()] += 1
    free = tokens - n_vision
    cuts = np.sort(rng.choice(free + 1, n_spans, replace=True))
    pos = 0
    prev = 0
    for s, c in zip(sizes, cuts):
        pos += c - prev
        prev = c
        tags[pos: pos + s] = 1
        pos += s
    return tags


def make_activations(rng, tokens, d_in, tags, c_text, c_vision, lo=30.0, hi=100.0,
                     dtype=np.float16):
    """N(0,1) activations; per-channel U(lo, hi) outlier scales on the text
    channels for text rows and on the vision channels for vision rows."""
    x = rng.standard_normal((tokens, d_in), dtype=np.float32)
    t_rows = tags == 0
    v_rows = ~t_rows
    if len(c_text):
        x[np.ix_(t_rows, c_text)] *= rng.uniform(lo, hi, len(c_text)).astype(np.float32)
    if len(c_vision):
        x[np.ix_(v_rows, c_vision)] *= rng.uniform(lo, hi, len(c_vision)).astype(np.float32)
    return x.astype(dtype)


def outlier_sets(rng, d_in, k):
    perm = rng.permutation(d_in)
    return np.sort(perm[:k]), np.sort(perm[k:2 * k])


def build_split_layer(mod, rng, spec: LayerSpec, col_max, c_text, c_vision, w=None,
                      factor_std=0.01):
    """Assemble a SplitLayer of module ``mod`` (the product package or the
    reference ``modquant``) with random-init weights and random low-rank
    factors of the reference default ranks (SVD anchoring is offline and
    does not change the work on the path)."""
    d_in, d_out = spec.d_in, spec.d_out
    c_text = np.asarray(c_text, np.int64)
    c_vision = np.asarray(c_vision, np.int64)
    mask = np.ones(d_in, bool)
    mask[c_text] = False
    mask[c_vision] = False
    c_main = np.flatnonzero(mask)
    part = mod.ChannelPartition(c_main, c_text, c_vision, d_in)
    if w is None:
        w = (rng.standard_normal((d_in, d_out), dtype=np.float32) * 0.02).astype(np.float64)
    init = mod.init_transform if hasattr(mod, "init_transform") else mod.transform.init_transform

    def tinit(idx):
        # transform.py:75-91 from the per-channel max |X| of the calibration batch
        cm = np.asarray(col_max, np.float64)[idx]
        if len(idx) == 0:
            return init(0, "diagonal", None)
        return init(len(idx), "diagonal", cm[np.newaxis, :])

    Granularity = mod.Granularity
    act = mod.QuantSpec(spec.abits, spec.a_sym, Granularity.PER_TOKEN)
    wsp = mod.QuantSpec(spec.wbits, True, Granularity.PER_CHANNEL)
    LRB = mod.LowRankBranch if hasattr(mod, "LowRankBranch") else mod.lowrank.LowRankBranch
    d_m = len(c_main)
    bs = bc = None
    if spec.r_cws:
        bs = LRB(rng.normal(0, factor_std, (d_m, spec.r_cws)),
                 rng.normal(0, factor_std, (spec.r_cws, d_out)), np.ones(spec.r_cws))
    if spec.r_mac:
        bc = LRB(rng.normal(0, factor_std, (d_m, spec.r_mac)),
                 rng.normal(0, factor_std, (spec.r_mac, d_out)), np.ones(spec.r_mac))
    SplitLayer = mod.SplitLayer if hasattr(mod, "SplitLayer") else mod.layer.SplitLayer
    return SplitLayer(
        partition=part, w_main=w[c_main], w_text=w[c_text], w_vision=w[c_vision],
        p_main=tinit(c_main), p_text=tinit(c_text), p_vision=tinit(c_vision),
        act_spec=act, weight_spec=wsp, branch_smooth=bs, branch_comp=bc,
        use_cws=bool(spec.r_cws), use_mac=bool(spec.r_mac),
    )


def config1(mod):
    """BASELINE config 1 (exact recipe above). Returns (layer, x fp32, tags)."""
    rng = np.random.default_rng(0)
    w = (rng.standard_normal((2048, 2048), dtype=np.float32) * np.float32(0.02)).astype(np.float64)
    x = rng.standard_normal((512, 2048), dtype=np.float32)
    tags = np.array([1] * 384 + [0] * 128, np.uint8)
    x[384:, 0:16] *= 50.0
    x[:384, 16:32] *= 50.0
    col_max = np.max(np.abs(x.astype(np.float64)), axis=0)
    spec = LayerSpec("c1", 2048, 2048, 16, 16, 16, 16)
    layer = build_split_layer(mod, np.random.default_rng(1), spec, col_max, np.arange(16),
                              np.arange(16, 32), w=w)
    return layer, x, tags


def model_specs(shape: dict, abits=4, wbits=4, a_sym=False):
    specs = []
    for name, d_in, d_out in projections(shape):
        k = shape["k_out"] or int(round(0.01 * d_in))
        d_m = d_in - 2 * k
        specs.append(LayerSpec(name, d_in, d_out, k, k, default_rank(0.02, d_m, d_out),
                               default_rank(0.03, d_m, d_out), abits, wbits, a_sym))
    return specs
