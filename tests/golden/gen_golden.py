#!/usr/bin/env python
"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):
    python tests/golden/gen_golden.py
It imports modquant read-only from /root/reference/pkg/src and writes small
.npz fixtures next to this script. The tests (and the GPU box) only read the
fixtures. Every fixture stores its inputs and the reference's outputs.
"""

from __future__ import annotations

import dataclasses
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import modquant as mq  # noqa: E402
from modquant import layer as L  # noqa: E402
from modquant import lowrank, mocd, quantizer as qz  # noqa: E402
from modquant.quantizer import Granularity, QuantSpec  # noqa: E402
from modquant.synth import SynthConfig, generate, generate_weight  # noqa: E402

GRAN = {"per_tensor": Granularity.PER_TENSOR, "per_channel": Granularity.PER_CHANNEL,
        "per_token": Granularity.PER_TOKEN}


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, os.path.getsize(path), "bytes")


def gen_quantizer():
    rng = np.random.default_rng(1234)
    out = {}
    cases = []
    for i, (bits, sym, gran, shape, scale) in enumerate([
        (4, False, "per_token", (17, 33), 1.0), (8, False, "per_token", (9, 64), 10.0),
        (2, False, "per_token", (5, 7), 0.1), (3, True, "per_token", (8, 40), 1.0),
        (8, True, "per_token", (6, 50), 100.0), (4, True, "per_channel", (40, 12), 0.02),
        (3, True, "per_channel", (31, 9), 1.0), (8, True, "per_channel", (64, 16), 1.0),
        (4, False, "per_channel", (20, 6), 1.0), (6, True, "per_tensor", (7, 7), 1.0),
    ]):
        m = rng.standard_normal(shape) * scale
        if i == 0:
            m[3] = 0.7  # constant row
            m[4] = 0.0  # all-zero row
        spec = QuantSpec(bits, sym, GRAN[gran])
        p = qz.compute_params(m, spec)
        out[f"m{i}"] = m
        out[f"s{i}"] = p.scales
        out[f"z{i}"] = p.zero_points
        out[f"fq{i}"] = qz.fake_quantize(m, p, spec)
        cases.append((bits, int(sym), list(GRAN).index(gran)))
    out["cases"] = np.array(cases, np.int64)
    # the reference tests' hand vector for round_half_away (test_quantizer.py:53-57)
    x = np.array([0.5, -0.5, 1.5, -1.5, 2.5, 0.4, -0.4, 0.49999999999999994, 2.5000000000000004])
    out["rha_x"] = x
    out["rha_y"] = qz.round_half_away(x)
    save("quantizer.npz", **out)


def layer_arrays(layer, prefix):
    p = layer.partition
    a = {
        f"{prefix}c_main": p.c_main, f"{prefix}c_text": p.c_text, f"{prefix}c_vision": p.c_vision,
        f"{prefix}w_main": layer.w_main, f"{prefix}w_text": layer.w_text,
        f"{prefix}w_vision": layer.w_vision,
        f"{prefix}log_main": layer.p_main.log_scale, f"{prefix}log_text": layer.p_text.log_scale,
        f"{prefix}log_vision": layer.p_vision.log_scale,
        f"{prefix}d_main": layer.p_main.scale, f"{prefix}d_text": layer.p_text.scale,
        f"{prefix}d_vision": layer.p_vision.scale,
        f"{prefix}specs": np.array([layer.act_spec.bits, layer.act_spec.symmetric,
                                    layer.weight_spec.bits, layer.weight_spec.symmetric,
                                    layer.use_cws, layer.use_mac, layer.aux_bits_floor], np.int64),
    }
    for name, br in (("bs", layer.branch_smooth), ("bc", layer.branch_comp)):
        if br is not None:
            a[f"{prefix}{name}_u"] = br.u_star
            a[f"{prefix}{name}_v"] = br.v_base
            a[f"{prefix}{name}_g"] = br.gate
    return a


def gen_layers():
    """Small layers in the reference's own test recipe (test_layer.py:27-45):
    synthetic planted-outlier batches, decaying-spectrum weights, MOCD
    partitions, build_layer with SVD-anchored CWS / MAC branches."""
    out = {}
    idx = 0
    for seed in range(4):
        batch = generate(SynthConfig(tokens_text=24, tokens_vision=16, dim=48,
                                     vision_outlier_channels=(1, 7),
                                     text_outlier_channels=(5, 30), seed=seed))
        w = generate_weight(48, 40, seed=seed + 10_000)
        part = mocd.build_partition(batch, mocd.MocdConfig(ratio_vision=2 / 48, ratio_text=2 / 48))
        for abits, wbits, asym, cws, mac in ((4, 4, False, True, True), (8, 4, False, True, True),
                                             (3, 3, False, True, False), (4, 4, True, False, True),
                                             (2, 3, False, False, False)):
            act = QuantSpec(abits, asym, Granularity.PER_TOKEN)
            wsp = QuantSpec(wbits, True, Granularity.PER_CHANNEL)
            layer = L.build_layer(w, batch, part, act, wsp, use_cws=cws, use_mac=mac)
            y, cache = L.forward_with_cache(layer, batch)
            pre = f"L{idx}_"
            out.update(layer_arrays(layer, pre))
            out[pre + "x"] = batch.data
            out[pre + "tags"] = batch.tags
            out[pre + "y"] = y
            out[pre + "x_hat"] = cache["m"]["x_hat"]
            if "mac" in cache:
                out[pre + "e_q"] = cache["mac"]["e_q"]
            if "t" in cache and cache["t"]["a"].shape[1]:
                out[pre + "a_t"] = cache["t"]["a"]
            out[pre + "y_ref"] = L.forward_reference(w, batch)
            idx += 1
    out["n_layers"] = np.array(idx)
    save("layers.npz", **out)


def gen_config1():
    """BASELINE config 1 built from its seeds (workloads.config1) through the
    reference; the fixture keeps a SHA-256 of the fp64 output plus samples."""
    import workloads as wl

    layer, x, tags = wl.config1(mq)
    batch = mq.ActivationBatch(x.astype(np.float64), tags)
    y = L.forward(layer, batch)
    rng = np.random.default_rng(0)
    rows = rng.integers(0, y.shape[0], 64)
    cols = rng.integers(0, y.shape[1], 64)
    save("config1.npz", sha256=np.frombuffer(hashlib.sha256(y.tobytes()).digest(), np.uint8),
         rows=rows, cols=cols, samples=y[rows, cols], rms=np.sqrt(np.mean(y ** 2)),
         shape=np.array(y.shape))


def gen_mocd():
    out = {}
    for seed in range(3):
        batch = generate(SynthConfig(seed=seed))
        cfg = mocd.MocdConfig(ratio_vision=2 / 64, ratio_text=2 / 64)
        part = mocd.build_partition(batch, cfg)
        cand = np.setdiff1d(np.arange(64), part.c_vision)
        ranks = mocd.percentile_rank(batch, cand)
        pre = f"s{seed}_"
        out[pre + "x"] = batch.data
        out[pre + "tags"] = batch.tags
        out[pre + "vscore"] = mocd.vision_score(batch)
        out[pre + "ranks"] = ranks
        out[pre + "tscore"] = mocd.text_score(ranks, 3, 50)
        out[pre + "c_text"] = part.c_text
        out[pre + "c_vision"] = part.c_vision
    # random batches with several clusters settings
    rng = np.random.default_rng(77)
    for i in range(3):
        data = rng.standard_normal((40, 24)) * rng.uniform(0.1, 5, 24)
        tags = np.array([0] * 30 + [1] * 10, np.uint8)
        batch = mq.ActivationBatch(data, tags)
        cfg = mocd.MocdConfig(ratio_vision=0.125, ratio_text=0.125, clusters_k=2 + i)
        part = mocd.build_partition(batch, cfg)
        pre = f"r{i}_"
        out[pre + "x"] = data
        out[pre + "tags"] = tags
        out[pre + "k"] = np.array(2 + i)
        out[pre + "c_text"] = part.c_text
        out[pre + "c_vision"] = part.c_vision
        cand = np.setdiff1d(np.arange(24), part.c_vision)
        out[pre + "tscore"] = mocd.text_score(mocd.percentile_rank(batch, cand), 2 + i, 50)
    save("mocd.npz", **out)


def gen_layer_dir():
    """A calibrated-layer directory written by the reference's save_layer
    (layer.py:284-322; manifest.json + SPQT dumps, tensor.py:118-135), plus an
    SPQT matrix and batch dump, and the layer's forward on its batch."""
    import shutil
    from modquant.tensor import save_tensor
    d = os.path.join(HERE, "layer_dir")
    shutil.rmtree(d, ignore_errors=True)
    batch = generate(SynthConfig(tokens_text=24, tokens_vision=16, dim=48, vision_outlier_channels=(1, 7),
                                 text_outlier_channels=(5, 30), seed=3))
    w = generate_weight(48, 40, seed=10_003)
    part = mocd.build_partition(batch, mocd.MocdConfig(ratio_vision=2 / 48, ratio_text=2 / 48))
    layer = L.build_layer(w, batch, part, QuantSpec(4, False, Granularity.PER_TOKEN),
                          QuantSpec(4, True, Granularity.PER_CHANNEL), use_cws=True, use_mac=True)
    L.save_layer(layer, d)
    save_tensor(os.path.join(d, "batch.spqt"), batch)
    save_tensor(os.path.join(d, "matrix.spqt"), w[:5, :7])
    np.save(os.path.join(d, "y_ref.npy"), L.forward(layer, batch))
    print("wrote", d, sorted(os.listdir(d)))


def gen_stability():
    """The reference's stability_report (calibrate.py:301-329) on a small
    planted batch: subset sizes, trials, the Jaccard mean / std per size."""
    from modquant.calibrate import stability_report
    batch = generate(SynthConfig(tokens_text=180, tokens_vision=120, dim=64, vision_outlier_channels=(2, 9),
                                 text_outlier_channels=(17, 40), vision_outlier_scale=1.6,
                                 text_instability=0.15, seed=5))
    cfg = mocd.MocdConfig(ratio_vision=4 / 64, ratio_text=4 / 64)
    sizes, ref_size, trials = [30, 90, 200], 260, 4
    rep = stability_report(batch, cfg, sizes, ref_size, trials, seed=2)
    save("stability.npz", x=batch.data, tags=batch.tags, sizes=np.array(sizes), ref_size=np.array(ref_size),
         trials=np.array(trials), ratios=np.array([cfg.ratio_vision, cfg.ratio_text]),
         mean=np.array([r["mean_jaccard"] for r in rep]), std=np.array([r["std_jaccard"] for r in rep]))


def gen_calib():
    """The reference's calibration caller (calibrate.py:146-270) on layers of
    the gen_layers recipe: loss + analytic straight-through gradient at the
    initial parameters, and a short calibrate() run (loss trace + final
    parameters)."""
    import importlib
    cal = importlib.import_module("modquant.calibrate")
    out = {}
    idx = 0
    for seed in range(2):
        batch = generate(SynthConfig(tokens_text=24, tokens_vision=16, dim=48,
                                     vision_outlier_channels=(1, 7),
                                     text_outlier_channels=(5, 30), seed=seed))
        w = generate_weight(48, 40, seed=seed + 10_000)
        part = mocd.build_partition(batch, mocd.MocdConfig(ratio_vision=2 / 48, ratio_text=2 / 48))
        for abits, wbits, cws, mac in ((4, 4, True, True), (3, 3, True, False), (4, 4, False, True)):
            act = QuantSpec(abits, False, Granularity.PER_TOKEN)
            wsp = QuantSpec(wbits, True, Granularity.PER_CHANNEL)
            layer = L.build_layer(w, batch, part, act, wsp, use_cws=cws, use_mac=mac)
            cfg = cal.CalibConfig(steps=6)
            segments = cal._param_layout(layer, cfg)
            y_ref = L.forward_reference(layer.full_weight(), batch)
            loss, grad = cal.analytic_gradient(layer, batch, segments, y_ref)
            final, trace = cal.calibrate(layer, batch, cfg)
            pre = f"C{idx}_"
            out.update(layer_arrays(layer, pre))
            out[pre + "x"] = batch.data
            out[pre + "tags"] = batch.tags
            out[pre + "loss"] = np.array(loss)
            out[pre + "grad"] = grad
            out[pre + "trace"] = np.array(trace.losses)
            out[pre + "theta"] = cal._initial_params(final, segments)
            idx += 1
    out["n_layers"] = np.array(idx)
    save("calib.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["quantizer", "layers", "config1", "mocd", "layer_dir", "stability", "calib"]
    for name in which:
        globals()["gen_" + name]()
