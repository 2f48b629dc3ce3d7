"""The calibration caller on the device (calib_gpu.py) against the
reference's own calibration (tests/golden/calib.npz and layers.npz, written
by gen_golden.py from modquant):

  * forward_with_cache: the fake-quantized activations (x_hat), MAC residual
    codes (e_q) and outlier-path activations are bit-identical (exact codes
    and scales from the K1 kernel); the output matches within fp64 summation
    order (cuBLAS vs OpenBLAS);
  * analytic_gradient (straight-through estimator, calibrate.py:146-222):
    loss and gradient at the reference's initial parameters;
  * calibrate(): the loss trace and the final parameters of a 6-step run.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _layer(d, p):
    import paper_2605_19929_b200 as pkg
    from paper_2605_19929_b200 import lowrank, transform as tr
    c_m, c_t, c_v = d[p + "c_main"], d[p + "c_text"], d[p + "c_vision"]
    dim = len(c_m) + len(c_t) + len(c_v)
    ab, a_sym, wb, w_sym, cws, mac, floor = (int(v) for v in d[p + "specs"])
    act = pkg.QuantSpec(ab, bool(a_sym), pkg.Granularity.PER_TOKEN)
    wsp = pkg.QuantSpec(wb, bool(w_sym), pkg.Granularity.PER_CHANNEL)
    br = lambda n: lowrank.LowRankBranch(d[p + n + "_u"], d[p + n + "_v"], d[p + n + "_g"]) \
        if p + n + "_u" in d else None
    tf = lambda k: tr.Transform(len(d[p + "log_" + k]), d[p + "log_" + k])
    layer = pkg.SplitLayer(pkg.ChannelPartition(c_m, c_t, c_v, dim), d[p + "w_main"], d[p + "w_text"],
                           d[p + "w_vision"], tf("main"), tf("text"), tf("vision"), act, wsp,
                           br("bs"), br("bc"), bool(cws), bool(mac), floor)
    return layer, pkg.ActivationBatch(d[p + "x"], d[p + "tags"])


@pytest.mark.parametrize("i", range(20))
def test_forward_with_cache_matches_reference(i):
    import paper_2605_19929_b200 as pkg
    d = np.load(os.path.join(GOLD, "layers.npz"))
    p = f"L{i}_"
    layer, batch = _layer(d, p)
    y, cache = pkg.forward_with_cache(layer, batch)
    np.testing.assert_array_equal(cache["m"]["x_hat"].cpu().numpy(), d[p + "x_hat"])
    if p + "e_q" in d:
        np.testing.assert_array_equal(cache["mac"]["e_q"].cpu().numpy(), d[p + "e_q"])
    if p + "a_t" in d:
        np.testing.assert_array_equal(cache["t"]["a"].cpu().numpy(), d[p + "a_t"])
    ref = d[p + "y"]
    np.testing.assert_allclose(y.cpu().numpy(), ref, rtol=0, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("i", range(6))
def test_analytic_gradient_matches_reference(i):
    from paper_2605_19929_b200 import calib_gpu as cg
    d = np.load(os.path.join(GOLD, "calib.npz"))
    p = f"C{i}_"
    layer, batch = _layer(d, p)
    cfg = cg.CalibConfig(steps=6)
    segments = cg._param_layout(layer, cfg)
    y_ref = batch.data @ layer.full_weight()
    loss, grad = cg.analytic_gradient(layer, batch, segments, y_ref)
    assert loss == pytest.approx(float(d[p + "loss"]), rel=1e-12)
    g_ref = d[p + "grad"]
    np.testing.assert_allclose(grad, g_ref, rtol=0, atol=1e-9 * np.abs(g_ref).max())


@pytest.mark.parametrize("i", range(6))
def test_calibrate_trace_matches_reference(i):
    import paper_2605_19929_b200 as pkg
    from paper_2605_19929_b200 import calib_gpu as cg
    d = np.load(os.path.join(GOLD, "calib.npz"))
    p = f"C{i}_"
    layer, batch = _layer(d, p)
    cfg = pkg.CalibConfig(steps=6)
    final, trace = pkg.calibrate(layer, batch, cfg)
    np.testing.assert_allclose(trace.losses, d[p + "trace"], rtol=1e-9)
    theta = cg._initial_params(final, cg._param_layout(final, cfg))
    np.testing.assert_allclose(theta, d[p + "theta"], rtol=0, atol=1e-9 * max(1.0, np.abs(d[p + "theta"]).max()))


def test_nonfinite_batch_raises():
    import paper_2605_19929_b200 as pkg
    d = np.load(os.path.join(GOLD, "calib.npz"))
    layer, batch = _layer(d, "C0_")
    x = batch.data.copy()
    x[3, 4] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        pkg.forward_with_cache(layer, pkg.ActivationBatch(x, batch.tags))
