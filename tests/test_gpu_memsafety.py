"""Memory-safety checks of every kernel family through the C-ABI (the pool's
GPUs do not run compute-sanitizer; these are its analogues):

  * guard bands (memcheck): the workspace, the output and the MOCD count
    buffers sit between 64 KB guard regions filled with a sentinel; no
    launch may write outside its buffer, or into y's padding columns
    (y_ld > d_out);
  * uninitialised reads (initcheck): the workspace is filled with 0x00, 0xFF
    and random bytes before the call; codes, accumulators and outputs must
    be bit-identical, so nothing reads workspace bytes it did not write;
  * out-of-row reads: x carries NaN in the padding columns past d_in
    (x_ld > d_in) and the forward must neither see them (no non-finite
    error) nor change its output;
  * repeatability (racecheck analogue): five runs bit-identical.
Regimes: K1 warp rows + tcgen05 split GEMM + LR1 (prefill), packed 4-bit
weights, K1 row groups + decode GEMVs, the fp32 / fp64 row-group K1, the
fp64 MAC pass (8-bit aux codes), swap-AB + split-K, and the MOCD kernels."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import workloads as wl  # noqa: E402

pytestmark = pytest.mark.gpu
GUARD = 1 << 16
SENT = 0xA5


def _layer(seed, T, d_in, d_out, k, r_s, r_c, abits=4):
    import paper_2605_19929_b200 as pkg
    from paper_2605_19929_b200 import runtime
    rng = np.random.default_rng(seed)
    tags = wl.tags_with_spans(rng, T, T // 4)
    c_t, c_v = wl.outlier_sets(rng, d_in, k)
    x = wl.make_activations(rng, T, d_in, tags, c_t, c_v, dtype=np.float32)
    layer = wl.build_split_layer(pkg, rng, wl.LayerSpec("m", d_in, d_out, k, k, r_s, r_c, abits, 4),
                                 np.max(np.abs(x), axis=0), c_t, c_v)
    return runtime.GpuLayer(layer, runtime.device()), x, tags


CASES = {  # name: (layer args, x dtype)
    "prefill_f16": ((1, 700, 512, 384, 16, 16, 16), torch.float16),
    "packed_w4_f16": ((2, 1200, 768, 256, 16, 8, 8), torch.float16),
    "decode_t3_f16": ((3, 3, 512, 256, 16, 8, 8), torch.float16),
    "decode_t40_swap_f16": ((4, 40, 640, 200, 16, 8, 8), torch.float16),
    "group_f32": ((5, 200, 384, 160, 8, 4, 6), torch.float32),
    "group_f64": ((6, 130, 256, 96, 8, 4, 6), torch.float64),
    "a8_mac_fp64_pass": ((7, 700, 640, 256, 32, 10, 15, 8), torch.float16),
}


def _run(gl, x, tags, dt, fill, ld_pad=8, raw=False):
    T, d_in = x.shape
    xd = torch.full((T, d_in + ld_pad), float("nan"), dtype=dt, device="cuda")
    xd[:, :d_in] = torch.from_numpy(x).to(dt).cuda()
    td = torch.from_numpy(tags).cuda()
    lay = gl.layout(T)
    n = int(lay.total_bytes)
    buf = torch.full((n + 2 * GUARD,), SENT, dtype=torch.uint8, device="cuda")
    ws = buf[GUARD:GUARD + n]
    if fill == "zero":
        ws.zero_()
    elif fill == "ones":
        ws.fill_(0xFF)
    else:
        ws.copy_(torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda"))
    y_ld = gl.d_out + 24
    if raw:  # the two raw planes are allocated by run(); the workspace guards still apply
        out = gl.run(xd[:, :d_in], td, raw=True, ws=ws).cpu().numpy()
    else:
        ybuf = torch.full((T * y_ld + 2 * GUARD // 4,), -7.25, dtype=torch.float32, device="cuda")
        yv = ybuf[GUARD // 4: GUARD // 4 + T * y_ld].view(T, y_ld)
        gl.run(xd[:, :d_in], td, y=yv[:, :gl.d_out], ws=ws)
        out = yv[:, :gl.d_out].cpu().numpy()
        pad = yv[:, gl.d_out:].cpu().numpy()
        assert np.all(pad == -7.25), "write into y's padding columns"
        yb = ybuf.cpu().numpy()
        assert np.all(yb[:GUARD // 4] == -7.25) and np.all(yb[GUARD // 4 + T * y_ld:] == -7.25), "y guard hit"
    torch.cuda.synchronize()
    b = buf.cpu().numpy()
    assert np.all(b[:GUARD] == SENT) and np.all(b[GUARD + n:] == SENT), "workspace guard hit"
    return out


@pytest.mark.parametrize("name", sorted(CASES))
def test_guards_and_uninitialised_workspace(name):
    args, dt = CASES[name]
    gl, x, tags = _layer(*args)
    outs = [_run(gl, x, tags, dt, fill) for fill in ("zero", "ones", "random")]
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])
    raws = [_run(gl, x, tags, dt, fill, raw=True) for fill in ("zero", "random")]
    np.testing.assert_array_equal(raws[1][0], raws[0][0])  # int32 main accumulators
    # repeatability
    for _ in range(3):
        np.testing.assert_array_equal(_run(gl, x, tags, dt, "random"), outs[0])


def test_mocd_guards():
    from paper_2605_19929_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(9)
    T, D = 3000, 96
    x = torch.from_numpy((rng.standard_normal((T, D)) * rng.uniform(0.1, 5, D)).astype(np.float16)).cuda()
    tags = rng.permutation(np.array([0] * 2200 + [1] * 800, np.uint8))
    td = torch.from_numpy(tags).cuda()
    rows = torch.from_numpy(np.flatnonzero(tags == 0).astype(np.int32)).cuda()
    nt = torch.tensor([rows.numel()], dtype=torch.int32, device="cuda")
    cand = torch.arange(3, D, dtype=torch.int32, device="cuda")
    n = rows.numel() * cand.numel()
    buf = torch.full((n + 2 * GUARD,), -23131, dtype=torch.int16, device="cuda")
    counts = buf[GUARD:GUARD + n]
    _lib.check(lib.splitq_mocd_rank_counts(x.data_ptr(), _lib.F16, D, rows.data_ptr(), nt.data_ptr(),
                                           rows.numel(), cand.data_ptr(), cand.numel(), counts.data_ptr(),
                                           None))
    vb = torch.full((D + 2 * 512,), -1.5, dtype=torch.float64, device="cuda")
    ab = torch.full((D + 2 * 512,), -1.5, dtype=torch.float64, device="cuda")
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    _lib.check(lib.splitq_mocd_absmax(x.data_ptr(), _lib.F16, D, td.data_ptr(), T, D, vb[512:512 + D].data_ptr(),
                                      ab[512:512 + D].data_ptr(), st.data_ptr(), None))
    torch.cuda.synchronize()
    b = buf.cpu().numpy()
    assert np.all(b[:GUARD] == -23131) and np.all(b[GUARD + n:] == -23131)
    for t in (vb, ab):
        h = t.cpu().numpy()
        assert np.all(h[:512] == -1.5) and np.all(h[512 + D:] == -1.5)
