"""GPU parity of the half-precision K1 path (csrc/k1w.cuh) against the oracle.

fp16 / bf16 inputs take the fp32-fast-path quantizer with the exact fp64
fallback; these cases push it where the fallback matters: exact .5 ties in
the main and MAC residual codes (half-integer inputs at unit smoothing),
constant and all-zero rows, rows far from zero (the fixed-point range
check), non-finite values and bad tags. Every case checks codes, scales and
zero points bit-exactly and the fp32 output within 1e-3 of the output RMS.
"""

import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import workloads as wl
from oracle import splitq_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _pkg():
    import paper_2605_19929_b200 as pkg
    return pkg


def _to_dev(x64, dt):
    """(device tensor of dtype dt, the exact float64 values it holds)."""
    t = torch.from_numpy(np.ascontiguousarray(x64, dtype=np.float32)).to(dt)
    return t.cuda(), t.double().numpy()


def _layer(rng, T, d_in, d_out, k_t, k_v, r_s, r_c, abits=4, a_sym=False, col_max=None, x=None,
           tags=None):
    pkg = _pkg()
    c_t, c_v = wl.outlier_sets(rng, d_in, max(k_t, k_v, 1))
    c_t, c_v = c_t[:k_t], c_v[:k_v]
    if col_max is None:
        col_max = np.max(np.abs(x), axis=0)
    spec = wl.LayerSpec("k1w", d_in, d_out, k_t, k_v, r_s, r_c, abits, 4, a_sym)
    return wl.build_split_layer(pkg, rng, spec, col_max, c_t, c_v), c_t, c_v


def _check(layer, xd, x64, tags):
    from paper_2605_19929_b200 import runtime
    L = orc.from_reference_layer(layer)
    act = orc.activation_codes(L, x64, tags)
    g = runtime.packed(layer)
    T = x64.shape[0]
    ws = g.workspace(T)
    td = torch.from_numpy(tags).cuda()
    y = g.run(xd, td, ws=ws).double().cpu().numpy()
    torch.cuda.synchronize()
    lay = g.layout(T)
    wsn = ws.cpu().numpy()

    def view(off, dt, n):
        return wsn[off: off + np.dtype(dt).itemsize * n].view(dt)

    def codes_of(off, ld, rows, cols, centered, zp, main):
        c = view(off, np.int8, rows * ld).reshape(rows, ld)
        if main and lay.main_natural:
            c = c[:, np.asarray(layer.partition.c_main)]
        c = c[:, :cols].astype(np.int64)
        return c + zp[:, None] if centered else (c & 0xFF)

    q, s, z = act["main"]
    zp = view(lay.zp_main, np.int32, T).astype(np.int64)
    np.testing.assert_array_equal(zp, z)
    np.testing.assert_array_equal(view(lay.s_main, np.float64, T), s)
    np.testing.assert_array_equal(codes_of(lay.a_main, lay.ld_main, T, q.shape[1],
                                           lay.code_centered_main, zp, True), q)
    for name, oa, os_, oz, ld in (("text", lay.a_text, lay.s_text, lay.zp_text, lay.ld_text),
                                  ("vision", lay.a_vision, lay.s_vision, lay.zp_vision,
                                   lay.ld_vision)):
        if name in act:
            q, s, z = act[name]
            zp = view(oz, np.int32, T).astype(np.int64)
            np.testing.assert_array_equal(zp, z)
            np.testing.assert_array_equal(view(os_, np.float64, T), s)
            np.testing.assert_array_equal(codes_of(oa, ld, T, q.shape[1], lay.code_centered_aux,
                                                   zp, False), q)
    if "mac" in act:
        q, s, z = act["mac"]
        n = q.shape[0]
        assert int(view(lay.n_text, np.int32, 1)[0]) == n
        rows = view(lay.text_rows, np.int32, n)  # slot -> row (claimed in any order)
        np.testing.assert_array_equal(np.sort(rows), act["text_rows"])
        order = np.argsort(rows, kind="stable")
        zp = view(lay.zp_mac, np.int32, n).astype(np.int64)
        np.testing.assert_array_equal(zp[order], z)
        np.testing.assert_array_equal(view(lay.s_mac, np.float64, n)[order], s)
        np.testing.assert_array_equal(codes_of(lay.a_mac, lay.ld_main, n, q.shape[1],
                                               lay.code_centered_aux, zp, True)[order], q)
    ref = orc.forward(L, x64, tags)
    rms = np.sqrt(np.mean(ref ** 2))
    err = np.max(np.abs(y - ref)) / rms
    assert err <= TOL, f"max err {err:.3e} x rms"


DTS = [torch.float16, torch.bfloat16]
SHAPES = {
    "c1_small": dict(T=256, d_in=512, d_out=384, k_t=16, k_v=16, r_s=16, r_c=16),
    "a8": dict(T=300, d_in=640, d_out=256, k_t=32, k_v=32, r_s=10, r_c=15, abits=8),
    "a3": dict(T=129, d_in=512, d_out=200, k_t=8, k_v=8, r_s=8, r_c=12, abits=3),
    "a2": dict(T=77, d_in=384, d_out=144, k_t=8, k_v=8, r_s=4, r_c=6, abits=2),
    "sym4": dict(T=200, d_in=512, d_out=256, k_t=16, k_v=16, r_s=8, r_c=8, a_sym=True),
    "sym8": dict(T=160, d_in=512, d_out=256, k_t=16, k_v=16, r_s=8, r_c=8, abits=8, a_sym=True),
    "no_outliers": dict(T=256, d_in=512, d_out=256, k_t=0, k_v=0, r_s=8, r_c=8),
    "no_lowrank": dict(T=256, d_in=512, d_out=256, k_t=16, k_v=16, r_s=0, r_c=0),
    "one_token": dict(T=1, d_in=256, d_out=128, k_t=4, k_v=4, r_s=4, r_c=4),
    "wide_cpt4": dict(T=96, d_in=8192, d_out=128, k_t=32, k_v=32, r_s=4, r_c=4),
    "wide_cpt3": dict(T=64, d_in=5376, d_out=96, k_t=20, k_v=20, r_s=4, r_c=4),
    "odd_chunks": dict(T=50, d_in=1048, d_out=64, k_t=8, k_v=8, r_s=4, r_c=4),
}


@pytest.fixture(params=[("1", "0", "0", "1"), ("1", "0", "1", "1"), ("1", "1", "0", "1"), ("8", "0", "0", "1"),
                        ("8", "0", "0", "0"), ("16", "0", "0", "1")],
                ids=["warp_rows", "warp_rows_prefetch", "warp_rows_sync", "cta8_rows", "cta8_rows_global_d",
                     "cta16_rows"],
                autouse=True)
def k1_row_group(request, monkeypatch):
    """Every case runs with one warp per row (prefill; plain, with loads one
    chunk ahead, with the per-round CTA barrier) and with 8- / 16-warp row
    groups (decode-sized calls; the smoothing factors staged in SMEM with
    the row, or read from the global table as for wide rows with many rows
    per CTA); the library reads SPLITQ_K1_WPR / _SYNC / _PF / _STAGE_D per
    call."""
    monkeypatch.setenv("SPLITQ_K1_WPR", request.param[0])
    monkeypatch.setenv("SPLITQ_K1_SYNC", request.param[1])
    monkeypatch.setenv("SPLITQ_K1_PF", request.param[2])
    monkeypatch.setenv("SPLITQ_K1_STAGE_D", request.param[3])


@pytest.mark.parametrize("dt", DTS, ids=["f16", "bf16"])
@pytest.mark.parametrize("name", sorted(SHAPES))
def test_half_input_parity(name, dt):
    sh = dict(SHAPES[name])
    rng = np.random.default_rng(zlib.crc32(name.encode()) + (7 if dt is torch.bfloat16 else 0))
    T, d_in = sh["T"], sh["d_in"]
    tags = wl.tags_with_spans(rng, T, T // 4)
    x = rng.standard_normal((T, d_in))
    x[:, rng.permutation(d_in)[:8]] *= rng.uniform(30, 100, 8)
    xd, x64 = _to_dev(x, dt)
    layer, _, _ = _layer(rng, x=x64, tags=tags, **sh)
    _check(layer, xd, x64, tags)


@pytest.mark.parametrize("abits,sym", [(4, False), (8, False), (3, False), (4, True), (2, False)])
def test_exact_ties(abits, sym):
    """Half-integer inputs at unit smoothing: z / S and the MAC residual hit
    .5 exactly for a large share of elements (the exact fallback path)."""
    rng = np.random.default_rng(100 + abits)
    T, d_in = 192, 1024
    lvl = (1 << abits) - 1
    x = rng.integers(0, 2 * lvl + 1, (T, d_in)) * 0.5  # 0, 0.5, ..., lvl
    x[:, 0] = 0.0
    x[:, 1] = lvl  # every row spans [0, lvl] -> S = 1 (asym) exactly
    x[T // 2:] -= lvl / 2.0
    tags = wl.tags_with_spans(rng, T, T // 3)
    xd, x64 = _to_dev(x, torch.float16)
    layer, _, _ = _layer(rng, T, d_in, 128, 16, 16, 4, 8, abits=abits, a_sym=sym,
                         col_max=np.ones(d_in))
    _check(layer, xd, x64, tags)


def test_special_rows():
    """Constant rows, all-zero rows, rows far from zero (fixed-point range
    fallback) and rows with a single huge value."""
    rng = np.random.default_rng(7)
    T, d_in = 64, 768
    x = rng.standard_normal((T, d_in))
    x[0] = 0.0
    x[1] = 3.0
    x[2] = -2.5
    x[3] = 1000.0 + rng.uniform(0, 0.5, d_in)  # all positive, narrow: |z / S| ~ 3e4
    x[4] = -20000.0 + rng.uniform(0, 1.0, d_in)  # |z / S| ~ 3e5
    x[5, 7] = 60000.0
    x[6] = rng.standard_normal(d_in) * 1e-4
    tags = np.zeros(T, np.uint8)
    tags[T // 2:] = 1
    for dt in DTS:
        xd, x64 = _to_dev(x, dt)
        layer, _, _ = _layer(rng, T, d_in, 64, 8, 8, 4, 4, col_max=np.ones(d_in))
        _check(layer, xd, x64, tags)


def test_nonfinite_and_tags():
    pkg = _pkg()
    rng = np.random.default_rng(9)
    T, d_in = 32, 512
    x = rng.standard_normal((T, d_in))
    tags = np.zeros(T, np.uint8)
    layer, c_t, _ = _layer(rng, T, d_in, 64, 8, 8, 4, 4, x=x, tags=tags)
    main_col = int(layer.partition.c_main[3])
    for dt in DTS:
        for col, val in ((main_col, np.nan), (main_col, np.inf), (main_col, -np.inf),
                         (int(c_t[0]), np.nan), (int(c_t[0]), -np.inf)):
            bad = x.copy()
            bad[5, col] = val
            xd, _ = _to_dev(bad, dt)
            with pytest.raises(ValueError, match="non-finite"):
                pkg.forward(layer, pkg.ActivationBatch(xd, torch.from_numpy(tags).cuda()))
        xd, _ = _to_dev(x, dt)
        bt = torch.from_numpy(tags.copy()).cuda()
        bt[3] = 7
        with pytest.raises(ValueError, match="tags"):
            pkg.forward(layer, pkg.ActivationBatch(xd, bt))
