"""torch.library custom ops over the C-ABI (paper_2605_19929_b200/ops.py):
identical results to the direct GpuLayer / quantize_rows calls, CUDA-graph
capture and replay, torch.library.opcheck, and status checking."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from test_gpu_forward import CASES, _case  # noqa: E402

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2605_19929_b200 import ops
    return ops


@pytest.mark.parametrize("name,x16", [("c1_small", False), ("f16_input", True), ("decode_t2", False)])
def test_forward_op_matches_run(name, x16):
    from paper_2605_19929_b200 import runtime
    ops = _ops()
    layer, x, tags = _case(**CASES[name])
    lid = ops.register_layer(layer)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(tags).cuda()
    ws = ops.workspace_for(lid, x.shape[0])
    for dt in (torch.float32, torch.float16):
        y = ops.forward(lid, xd, td, ws, out_dtype=dt)
        ops.check_status(ws)
        ref = runtime.packed(layer).run(xd, td, out_dtype=dt)
        assert y.dtype == dt and y.shape == ref.shape
        np.testing.assert_array_equal(y.cpu().numpy(), ref.cpu().numpy())


def test_forward_op_cuda_graph():
    """The op launches without host synchronisation: capture it in a CUDA
    graph, replay on new inputs written into the captured buffers."""
    ops = _ops()
    layer, x, tags = _case(**CASES["c1_small"])
    lid = ops.register_layer(layer)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(tags).cuda()
    ws = ops.workspace_for(lid, x.shape[0])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up outside the capture (attributes, first-call set-up)
        for _ in range(2):
            ops.forward(lid, xd, td, ws)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        y_graph = ops.forward(lid, xd, td, ws)
    rng = np.random.default_rng(5)
    for _ in range(3):
        x2 = (x * rng.uniform(0.5, 2.0)).astype(x.dtype)
        xd.copy_(torch.from_numpy(x2).cuda())
        g.replay()
        torch.cuda.synchronize()
        ops.check_status(ws)
        eager = ops.forward(lid, xd, td, ops.workspace_for(lid, x.shape[0]))
        np.testing.assert_array_equal(y_graph.cpu().numpy(), eager.cpu().numpy())


def test_forward_op_opcheck():
    ops = _ops()
    layer, x, tags = _case(**CASES["tiny_dout"])
    lid = ops.register_layer(layer)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(tags).cuda()
    ws = ops.workspace_for(lid, x.shape[0])
    torch.library.opcheck(torch.ops.splitq.forward.default, (xd, td, ws, lid, 0),
                          test_utils=("test_schema", "test_faketensor"))


def test_forward_op_status_raises():
    ops = _ops()
    layer, x, tags = _case(**CASES["tiny_dout"])
    lid = ops.register_layer(layer)
    bad = x.copy()
    bad[2, 3] = np.nan
    ws = ops.workspace_for(lid, x.shape[0])
    ops.forward(lid, torch.from_numpy(bad).cuda(), torch.from_numpy(tags).cuda(), ws)
    with pytest.raises(ValueError, match="non-finite"):
        ops.check_status(ws)


def test_quantize_op_matches_reference_codes():
    from oracle import splitq_oracle as orc
    _ops()
    rng = np.random.default_rng(3)
    m = rng.standard_normal((41, 300)) * rng.uniform(0.1, 10, (41, 1))
    xd = torch.from_numpy(m).cuda()
    for bits, sym in ((4, False), (8, False), (3, True)):
        codes, s, z, st = torch.ops.splitq.quantize_per_token(xd, bits, sym)
        assert int(st[0]) == 0
        qo, so, zo = orc.codes(m, orc.Spec(bits, sym, orc.PER_TOKEN))
        c = codes[:, :300].cpu().numpy().astype(np.int64)
        zz = z.cpu().numpy().astype(np.int64)
        q = c + zz[:, None] if (sym or bits <= 7) else (c & 0xFF)
        np.testing.assert_array_equal(q, qo)
        np.testing.assert_array_equal(s.cpu().numpy(), so)
        np.testing.assert_array_equal(zz, zo)
