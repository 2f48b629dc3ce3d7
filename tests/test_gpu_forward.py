"""GPU parity of the split-linear forward against the CPU oracle.

Bars (BASELINE.json north star):
  * activation codes, scales and zero points: bit-exact (scales as fp64);
  * int32 main / text / vision accumulators: bit-exact;
  * fp32 output: max |y_gpu - y_ref| <= 1e-3 * rms(y_ref).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import workloads as wl
from oracle import splitq_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-3  # of the output RMS (north star)


def _pkg():
    import paper_2605_19929_b200 as pkg
    return pkg


def _case(seed, T, d_in, d_out, k_t, k_v, r_s, r_c, abits=4, wbits=4, a_sym=False,
          n_vision=None, x_dtype=np.float32, scale=(30.0, 100.0)):
    pkg = _pkg()
    rng = np.random.default_rng(seed)
    if n_vision is None:
        n_vision = T // 4
    tags = wl.tags_with_spans(rng, T, n_vision)
    c_t, c_v = wl.outlier_sets(rng, d_in, max(k_t, k_v))
    c_t, c_v = c_t[:k_t], c_v[:k_v]
    x = wl.make_activations(rng, T, d_in, tags, c_t, c_v, *scale, dtype=x_dtype)
    col_max = np.max(np.abs(x.astype(np.float64)), axis=0)
    spec = wl.LayerSpec("t", d_in, d_out, k_t, k_v, r_s, r_c, abits, wbits, a_sym)
    layer = wl.build_split_layer(pkg, rng, spec, col_max, c_t, c_v)
    return layer, x, tags


def _ws_view(ws, off, dtype, count):
    nbytes = np.dtype(dtype).itemsize * count
    return ws[off: off + nbytes].cpu().numpy().view(dtype)


def _run_gpu(layer, x, tags, raw=False):
    from paper_2605_19929_b200 import runtime
    g = runtime.packed(layer)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(tags).cuda()
    ws = g.workspace(x.shape[0])
    y = g.run(xd, td, raw=raw, ws=ws)
    torch.cuda.synchronize()
    return g, ws, y


def _check_codes(layer, x, tags):
    L = orc.from_reference_layer(layer)
    act = orc.activation_codes(L, x.astype(np.float64), tags)
    g, ws, _ = _run_gpu(layer, x, tags)
    lay = g.layout(x.shape[0])
    T = x.shape[0]
    cen_m, cen_a = lay.code_centered_main, lay.code_centered_aux

    def codes_of(off, ld, rows, cols, centered, zp, main=False):
        c = _ws_view(ws, off, np.int8, rows * ld).reshape(rows, ld)
        if main and lay.main_natural:  # natural channel order -> the reference's C_m order
            c = c[:, np.asarray(layer.partition.c_main)]
        c = c[:, :cols].astype(np.int64)
        return c + zp[:, None] if centered else (c & 0xFF)

    q, s, z = act["main"]
    zp = _ws_view(ws, lay.zp_main, np.int32, T).astype(np.int64)
    np.testing.assert_array_equal(zp, z)
    np.testing.assert_array_equal(_ws_view(ws, lay.s_main, np.float64, T), s)
    np.testing.assert_array_equal(codes_of(lay.a_main, lay.ld_main, T, q.shape[1], cen_m, zp, main=True), q)
    for name, off_a, off_s, off_z, ld in (("text", lay.a_text, lay.s_text, lay.zp_text, lay.ld_text),
                                          ("vision", lay.a_vision, lay.s_vision, lay.zp_vision,
                                           lay.ld_vision)):
        if name not in act:
            continue
        q, s, z = act[name]
        zp = _ws_view(ws, off_z, np.int32, T).astype(np.int64)
        np.testing.assert_array_equal(zp, z)
        np.testing.assert_array_equal(_ws_view(ws, off_s, np.float64, T), s)
        np.testing.assert_array_equal(codes_of(off_a, ld, T, q.shape[1], cen_a, zp), q)
    if "mac" in act:
        q, s, z = act["mac"]
        n = q.shape[0]
        assert int(_ws_view(ws, lay.n_text, np.int32, 1)[0]) == n
        # compact MAC rows may be claimed in any order: slot -> row map
        rows = _ws_view(ws, lay.text_rows, np.int32, n)
        np.testing.assert_array_equal(np.sort(rows), act["text_rows"])
        order = np.argsort(rows, kind="stable")
        zp = _ws_view(ws, lay.zp_mac, np.int32, n).astype(np.int64)[order]
        np.testing.assert_array_equal(zp, z)
        np.testing.assert_array_equal(_ws_view(ws, lay.s_mac, np.float64, n)[order], s)
        codes = codes_of(lay.a_mac, lay.ld_main, n, q.shape[1], cen_a,
                         _ws_view(ws, lay.zp_mac, np.int32, n).astype(np.int64), main=True)
        np.testing.assert_array_equal(codes[order], q)


def _check_acc(layer, x, tags):
    L = orc.from_reference_layer(layer)
    acc = orc.accumulators(L, x.astype(np.float64), tags)
    act = orc.activation_codes(L, x.astype(np.float64), tags)
    w = orc.weight_codes(L)
    g, _, y = _run_gpu(layer, x, tags, raw=True)
    lay = g.layout(x.shape[0])
    planes = y.cpu().numpy().astype(np.int64)
    T = x.shape[0]

    def expect(name, centered):
        # u8 (non-centred) codes: the tensor core accumulates q * w; the zero
        # point term zp * colsum(w) is removed in the epilogue
        if centered:
            return acc[name]
        return acc[name] + act[name][2][:, None] * w[name][0].sum(axis=0)[None, :]

    # the int32 main-channel accumulator is bit-exact (north-star bar); the
    # outlier / low-rank branches share the fp32 auxiliary accumulator and are
    # covered by the output tolerance test
    np.testing.assert_array_equal(planes[0], expect("main", lay.code_centered_main))
    assert planes.shape == (2, T, L.d_out)


def _check_out(layer, x, tags, out_dtype=None):
    pkg = _pkg()
    L = orc.from_reference_layer(layer)
    ref = orc.forward(L, x.astype(np.float64), tags)
    batch = pkg.ActivationBatch(torch.from_numpy(np.ascontiguousarray(x)).cuda(),
                                torch.from_numpy(tags).cuda())
    y = pkg.forward(layer, batch, out_dtype=out_dtype).double().cpu().numpy()
    rms = np.sqrt(np.mean(ref ** 2))
    if out_dtype in (None, torch.float32):
        err = np.max(np.abs(y - ref)) / rms
        assert err <= TOL, f"max err {err:.3e} x rms"
        return err
    # half-precision storage: the fp32 result within TOL, then one rounding of
    # the output type (unit roundoff 2^-11 for fp16, 2^-8 for bf16; F11)
    u = 2.0 ** -11 if out_dtype == torch.float16 else 2.0 ** -8
    excess = np.abs(y - ref) - u * np.abs(ref)
    err = np.max(excess) / rms
    assert err <= TOL, f"max err beyond output rounding {err:.3e} x rms"
    return err


CASES = {
    "c1_small": dict(seed=1, T=256, d_in=512, d_out=384, k_t=16, k_v=16, r_s=16, r_c=16),
    "a8w4": dict(seed=2, T=300, d_in=640, d_out=256, k_t=32, k_v=32, r_s=10, r_c=15, abits=8),
    "a3w3": dict(seed=3, T=129, d_in=512, d_out=200, k_t=8, k_v=8, r_s=8, r_c=12, abits=3, wbits=3),
    "a2w3": dict(seed=4, T=77, d_in=384, d_out=144, k_t=8, k_v=8, r_s=4, r_c=6, abits=2, wbits=3),
    "sym_a4": dict(seed=5, T=200, d_in=512, d_out=256, k_t=16, k_v=16, r_s=8, r_c=8, a_sym=True),
    "sym_a8": dict(seed=6, T=160, d_in=512, d_out=256, k_t=16, k_v=16, r_s=8, r_c=8, abits=8,
                   a_sym=True),
    "no_lowrank": dict(seed=7, T=256, d_in=512, d_out=512, k_t=16, k_v=16, r_s=0, r_c=0),
    "cws_only": dict(seed=8, T=256, d_in=512, d_out=256, k_t=16, k_v=16, r_s=12, r_c=0),
    "mac_only": dict(seed=9, T=256, d_in=512, d_out=256, k_t=16, k_v=16, r_s=0, r_c=12),
    "no_outliers": dict(seed=10, T=256, d_in=512, d_out=256, k_t=0, k_v=0, r_s=8, r_c=8),
    "all_vision": dict(seed=11, T=200, d_in=512, d_out=256, k_t=16, k_v=16, r_s=8, r_c=8,
                       n_vision=200),
    "all_text": dict(seed=12, T=200, d_in=512, d_out=256, k_t=16, k_v=16, r_s=8, r_c=8,
                     n_vision=0),
    "one_token": dict(seed=13, T=1, d_in=256, d_out=128, k_t=4, k_v=4, r_s=4, r_c=4, n_vision=0),
    "k110_down": dict(seed=14, T=300, d_in=2048, d_out=256, k_t=110, k_v=110, r_s=20, r_c=30),
    "f16_input": dict(seed=15, T=256, d_in=768, d_out=512, k_t=32, k_v=32, r_s=16, r_c=16,
                      x_dtype=np.float16),
    "f64_input": dict(seed=16, T=128, d_in=512, d_out=256, k_t=16, k_v=16, r_s=8, r_c=8,
                      x_dtype=np.float64),
    "tiny_dout": dict(seed=17, T=64, d_in=128, d_out=12, k_t=4, k_v=4, r_s=2, r_c=3),
    # >= 64 n-tiles: m-fastest tile groups (G2Params.tile_gm)
    "wide_n": dict(seed=27, T=700, d_in=256, d_out=10400, k_t=8, k_v=8, r_s=8, r_c=8),
    # the reference defaults: A8 asym PER_TOKEN x W8 sym PER_CHANNEL (layer.py:40-41)
    "a8w8_default": dict(seed=28, T=300, d_in=640, d_out=256, k_t=32, k_v=32, r_s=10, r_c=15, abits=8,
                         wbits=8),
    "decode_t3_a8w8": dict(seed=29, T=3, d_in=512, d_out=256, k_t=16, k_v=16, r_s=8, r_c=8, abits=8,
                           wbits=8, n_vision=1),
    # decode-sized calls (<= 8 rows): the CUDA-core GEMV kernels
    "decode_t2": dict(seed=18, T=2, d_in=512, d_out=384, k_t=16, k_v=16, r_s=16, r_c=16, n_vision=0),
    "decode_t5_a8": dict(seed=19, T=5, d_in=640, d_out=256, k_t=32, k_v=32, r_s=10, r_c=15, abits=8,
                         n_vision=2),
    "decode_t8_a3w3": dict(seed=20, T=8, d_in=384, d_out=200, k_t=8, k_v=8, r_s=8, r_c=12, abits=3,
                           wbits=3, n_vision=3),
    "decode_t7_ld16": dict(seed=21, T=7, d_in=400, d_out=130, k_t=8, k_v=8, r_s=6, r_c=5, n_vision=1),
    "decode_t3_sym": dict(seed=22, T=3, d_in=512, d_out=256, k_t=16, k_v=16, r_s=8, r_c=8, a_sym=True,
                          n_vision=1),
    "decode_t4_k4096": dict(seed=23, T=4, d_in=4096, d_out=256, k_t=64, k_v=64, r_s=24, r_c=24,
                            n_vision=1),
    # 9..32 rows: 2 or 4 MMA n-tiles of 8 rows
    "decode_t16": dict(seed=24, T=16, d_in=512, d_out=384, k_t=16, k_v=16, r_s=16, r_c=16, n_vision=3),
    "decode_t27_a8": dict(seed=25, T=27, d_in=640, d_out=200, k_t=32, k_v=32, r_s=10, r_c=15, abits=8,
                          n_vision=5),
    "decode_t32_a3w3": dict(seed=26, T=32, d_in=2048, d_out=256, k_t=8, k_v=8, r_s=8, r_c=12, abits=3,
                            wbits=3, n_vision=0),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_codes_bit_exact(name):
    layer, x, tags = _case(**CASES[name])
    _check_codes(layer, x, tags)


@pytest.mark.parametrize("name", sorted(CASES))
def test_accumulators_bit_exact(name):
    layer, x, tags = _case(**CASES[name])
    _check_acc(layer, x, tags)


@pytest.mark.parametrize("name", sorted(CASES))
def test_output_within_tolerance(name):
    layer, x, tags = _case(**CASES[name])
    _check_out(layer, x, tags)


@pytest.mark.parametrize("dt", ["float16", "bfloat16"])
def test_half_outputs(dt):
    layer, x, tags = _case(**CASES["c1_small"])
    _check_out(layer, x, tags, out_dtype=getattr(torch, dt))


def test_config1_full():
    """BASELINE config 1: codes, accumulators and output vs the oracle."""
    pkg = _pkg()
    layer, x, tags = wl.config1(pkg)
    _check_codes(layer, x, tags)
    _check_acc(layer, x, tags)
    err = _check_out(layer, x, tags)
    assert err < 1e-4


def test_numpy_dropin_returns_float64():
    pkg = _pkg()
    layer, x, tags = _case(**CASES["c1_small"])
    batch = pkg.ActivationBatch(x.astype(np.float64), tags)
    y = pkg.forward(layer, batch)
    assert isinstance(y, np.ndarray) and y.dtype == np.float64
    ref = orc.forward(orc.from_reference_layer(layer), x.astype(np.float64), tags)
    assert np.max(np.abs(y - ref)) <= TOL * np.sqrt(np.mean(ref ** 2))


def test_mac_locality_bit_exact():
    """Vision rows are bit-identical with MAC on vs off (test_layer.py:87-99)."""
    import dataclasses
    pkg = _pkg()
    layer, x, tags = _case(**CASES["c1_small"])
    off = dataclasses.replace(layer, use_mac=False)
    xb = torch.from_numpy(x).cuda()
    tb = torch.from_numpy(tags).cuda()
    y_on = pkg.forward(layer, pkg.ActivationBatch(xb, tb)).cpu().numpy()
    y_off = pkg.forward(off, pkg.ActivationBatch(xb, tb)).cpu().numpy()
    v = tags == 1
    np.testing.assert_array_equal(y_on[v], y_off[v])
    assert np.any(y_on[~v] != y_off[~v])


def test_data_errors_raise_valueerror():
    pkg = _pkg()
    layer, x, tags = _case(**CASES["tiny_dout"])
    bad = x.copy()
    bad[3, 5] = np.inf
    xb = torch.from_numpy(bad).cuda()
    with pytest.raises(ValueError, match="non-finite"):
        pkg.forward(layer, pkg.ActivationBatch(xb, torch.from_numpy(tags).cuda()))
    bad_tags = torch.from_numpy(tags.copy()).cuda()
    bad_tags[0] = 2
    with pytest.raises(ValueError, match="tags"):
        pkg.forward(layer, pkg.ActivationBatch(torch.from_numpy(x).cuda(), bad_tags))
    with pytest.raises(ValueError, match="width"):
        pkg.forward(layer, pkg.ActivationBatch(torch.from_numpy(x[:, :-1].copy()).cuda(),
                                               torch.from_numpy(tags).cuda()))


def test_unsupported_specs_raise():
    import dataclasses
    pkg = _pkg()
    layer, x, tags = _case(**CASES["tiny_dout"])
    for spec in (pkg.QuantSpec(None, False, pkg.Granularity.PER_TOKEN),
                 pkg.QuantSpec(16, False, pkg.Granularity.PER_TOKEN)):
        bad = dataclasses.replace(layer, act_spec=spec)
        with pytest.raises(ValueError):
            pkg.forward(bad, pkg.ActivationBatch(x.astype(np.float64), tags))


def test_quantize_rows_matches_oracle():
    pkg = _pkg()
    rng = np.random.default_rng(21)
    m = rng.standard_normal((37, 1000)) * rng.uniform(0.01, 100, (37, 1))
    m[5] = 0.7  # constant row
    m[6] = 0.0  # all-zero row
    for bits, sym in ((4, False), (8, False), (2, False), (8, True), (3, True)):
        spec = pkg.QuantSpec(bits, sym, pkg.Granularity.PER_TOKEN)
        q, p = pkg.quantize_per_token(m, spec)
        qo, so, zo = orc.codes(m, orc.Spec(bits, sym, orc.PER_TOKEN))
        np.testing.assert_array_equal(q, qo)
        np.testing.assert_array_equal(p.scales, so)
        np.testing.assert_array_equal(p.zero_points, zo)


@pytest.mark.parametrize("name", ["c1_small", "a3w3", "a8w4", "k110_down", "decode_t2", "decode_t4_k4096",
                                  "decode_t16", "decode_t27_a8"])
def test_packed_weights_match_int8_weights(name):
    """The main GEMM streams 4-bit packed weight codes (unpacked in SMEM);
    its raw int32 accumulators and outputs equal those of the int8 copy."""
    from paper_2605_19929_b200 import runtime
    layer, x, tags = _case(**CASES[name])
    g = runtime.packed(layer)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(tags).cuda()
    # main int32 accumulators bit-exact; the fp32 auxiliary plane and the
    # outputs agree to fp32 rounding (split-K sums them in any order)
    a = g.run(xd, td, raw=True)
    b = g.run(xd, td, raw=True, unpacked=True)
    np.testing.assert_array_equal(a[0].cpu().numpy(), b[0].cpu().numpy())
    fa, fb = a[1].view(torch.float32).cpu().numpy(), b[1].view(torch.float32).cpu().numpy()
    np.testing.assert_allclose(fa, fb, rtol=1e-5, atol=1e-6 * np.abs(fb).max())
    ya = g.run(xd, td).cpu().numpy()
    yb = g.run(xd, td, unpacked=True).cpu().numpy()
    np.testing.assert_allclose(ya, yb, rtol=1e-5, atol=1e-5 * np.abs(yb).max())


@pytest.mark.parametrize("name", ["decode_t16", "decode_t27_a8", "decode_t32_a3w3"])
def test_gemv_multi_tile(name, monkeypatch):
    """9..32-row calls forced onto the GEMV kernels (2 / 4 MMA n-tiles; by
    default such calls take the tcgen05 swap-AB path): codes, int32
    accumulators and outputs against the oracle."""
    monkeypatch.setenv("SPLITQ_GEMV_MAX_ROWS", "32")
    layer, x, tags = _case(**CASES[name])
    _check_acc(layer, x, tags)
    _check_out(layer, x, tags)


@pytest.mark.parametrize("ksplit", ["1", "3"])
@pytest.mark.parametrize("name", ["decode_t2", "decode_t4_k4096", "decode_t16", "decode_t5_a8"])
def test_gemv_lr1_k_split(name, ksplit, monkeypatch):
    """The decode low-rank first stage with K split over CTAs (integer
    atomics, last-arriving CTA applies the epilogue) and unsplit: LR1
    outputs feed the aux operand, so the outputs and the int32 main
    accumulators must match the oracle either way."""
    monkeypatch.setenv("SPLITQ_GV_KSPLIT", ksplit)
    layer, x, tags = _case(**CASES[name])
    _check_acc(layer, x, tags)
    _check_out(layer, x, tags)


def test_run_validates_buffers():
    """GpuLayer.run rejects mismatched tags / outputs / devices before launching."""
    from paper_2605_19929_b200 import runtime
    layer, x, tags = _case(**CASES["tiny_dout"])
    g = runtime.packed(layer)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(tags).cuda()
    with pytest.raises(ValueError, match="tags length"):
        g.run(xd, td[:-1])
    with pytest.raises(ValueError, match="y must be"):
        g.run(xd, td, y=torch.empty((x.shape[0] - 1, g.d_out), device="cuda"))
    with pytest.raises(ValueError, match="y must be"):
        g.run(xd, td, y=torch.empty((x.shape[0], g.d_out)))
    with pytest.raises(ValueError, match="must be on"):
        g.run(xd.cpu(), td)
    y = g.run(xd, td)
    assert y.shape == (x.shape[0], g.d_out)


def test_packed_cache_sees_inplace_edits():
    """An in-place edit of the layer's scales / gates re-packs it."""
    from paper_2605_19929_b200 import runtime
    layer, x, tags = _case(**CASES["tiny_dout"])
    g1 = runtime.packed(layer)
    assert runtime.packed(layer) is g1
    layer.branch_smooth.gate[0] *= 0.5
    assert runtime.packed(layer) is not g1


@pytest.mark.parametrize("name", ["c1_small", "no_lowrank", "no_outliers", "f16_input", "wide_n", "k110_down",
                                  "sym_a4", "a3w3"])
@pytest.mark.parametrize("dt", ["float32", "float16"])
def test_fast_epilogue_bit_identical(name, dt, monkeypatch):
    """The split GEMM's fast epilogue (column constants from SMEM, packed
    fp32 math, magic-number int -> float) keeps the slow epilogue's rounding
    order: outputs bit-identical (SPLITQ_EPI_SLOW=1 selects the slow one)."""
    from paper_2605_19929_b200 import runtime
    c = dict(CASES[name])
    c["T"] = max(c["T"], 2100)  # the tcgen05 prefill path
    layer, x, tags = _case(**c)
    g = runtime.packed(layer)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(tags).cuda()
    a = g.run(xd, td, out_dtype=getattr(torch, dt)).cpu().numpy()
    monkeypatch.setenv("SPLITQ_EPI_SLOW", "1")
    b = g.run(xd, td, out_dtype=getattr(torch, dt)).cpu().numpy()
    np.testing.assert_array_equal(a, b)


def test_concurrent_calls_share_a_layer():
    """Host threads calling one layer on their own streams, each with its own
    workspace (GpuLayer.run's cached workspace is per layer; the prefill
    LR1 fork / join uses per-layer events and a side stream): every call's
    output equals the serial one."""
    import threading
    from paper_2605_19929_b200 import runtime
    layer, x, tags = _case(**CASES["c1_small"])
    g = runtime.packed(layer)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(tags).cuda()
    ref = g.run(xd, td).cpu().numpy()
    outs, errs = [None] * 4, []

    def work(i):
        try:
            s = torch.cuda.Stream()
            ws = torch.empty(int(g.layout(x.shape[0]).total_bytes), dtype=torch.uint8, device="cuda")
            torch.cuda.synchronize()
            with torch.cuda.stream(s):
                ys = [g.run(xd, td, ws=ws) for _ in range(8)]
            s.synchronize()
            outs[i] = [y.cpu().numpy() for y in ys]
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for o in outs:
        for y in o:
            np.testing.assert_array_equal(y, ref)
