"""The product's offline layer builder against layers the reference built
(tests/golden/layers.npz, written by gen_golden.py from modquant's own
build_layer, layer.py:185-232): the same weights, batch and partition give a
bit-identical SplitLayer -- smoothing transforms (transform.py:75-91), the
SVD-anchored CWS / MAC branches (lowrank.py:26-85) and the split weights.
The GPU variant takes the column max |X| from the device statistic
(mocd_gpu.channel_absmax) instead of the host reduction."""

import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "layers.npz"))
N = int(G["n_layers"])


def _inputs(i):
    import paper_2605_19929_b200 as pkg
    p = f"L{i}_"
    c_m, c_t, c_v = G[p + "c_main"], G[p + "c_text"], G[p + "c_vision"]
    dim = len(c_m) + len(c_t) + len(c_v)
    wm = G[p + "w_main"]
    w = np.empty((dim, wm.shape[1]))
    w[c_m], w[c_t], w[c_v] = wm, G[p + "w_text"], G[p + "w_vision"]
    ab, a_sym, wb, w_sym, cws, mac, _floor = (int(v) for v in G[p + "specs"])
    act = pkg.QuantSpec(ab, bool(a_sym), pkg.Granularity.PER_TOKEN)
    wsp = pkg.QuantSpec(wb, bool(w_sym), pkg.Granularity.PER_CHANNEL)
    part = pkg.ChannelPartition(c_m, c_t, c_v, dim)
    batch = pkg.ActivationBatch(G[p + "x"], G[p + "tags"])
    return pkg, w, batch, part, act, wsp, bool(cws), bool(mac)


def _compare(layer, i):
    p = f"L{i}_"
    for got, key in ((layer.w_main, "w_main"), (layer.w_text, "w_text"), (layer.w_vision, "w_vision"),
                     (layer.p_main.log_scale, "log_main"), (layer.p_text.log_scale, "log_text"),
                     (layer.p_vision.log_scale, "log_vision"), (layer.p_main.scale, "d_main"),
                     (layer.p_text.scale, "d_text"), (layer.p_vision.scale, "d_vision")):
        np.testing.assert_array_equal(np.asarray(got), G[p + key], err_msg=key)
    for name, br in (("bs", layer.branch_smooth), ("bc", layer.branch_comp)):
        if p + name + "_u" in G:
            assert br is not None, name
            np.testing.assert_array_equal(br.u_star, G[p + name + "_u"])
            np.testing.assert_array_equal(br.v_base, G[p + name + "_v"])
            np.testing.assert_array_equal(br.gate, G[p + name + "_g"])
        else:
            assert br is None, name


@pytest.mark.parametrize("i", range(N))
def test_build_layer_matches_reference(i):
    pkg, w, batch, part, act, wsp, cws, mac = _inputs(i)
    layer = pkg.build_layer(w, batch, part, act, wsp, use_cws=cws, use_mac=mac)
    _compare(layer, i)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(0, N, 3))
def test_build_layer_with_device_col_max(i):
    from paper_2605_19929_b200 import mocd_gpu
    pkg, w, batch, part, act, wsp, cws, mac = _inputs(i)
    col_max = mocd_gpu.channel_absmax(batch)
    np.testing.assert_array_equal(col_max, np.max(np.abs(batch.data), axis=0))
    layer = pkg.build_layer(w, batch, part, act, wsp, use_cws=cws, use_mac=mac, col_max=col_max)
    _compare(layer, i)
