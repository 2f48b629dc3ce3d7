"""The token-sharded forward (rows are independent, no collective
on the path) with the product's kernels on every rank: world_size 2 and 3 on
one GPU, each rank running GpuLayer.run (the C-ABI splitq_forward) on its
token_shard rows, the shards gathered with parallel.gather_rows over gloo
(host copies). The gathered int32 main accumulators equal the
single-process run bit for bit, and the outputs are within the north-star
bar (1e-3 of the output RMS) of the oracle.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
T, D_IN, D_OUT = 1500, 512, 384


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    import paper_2605_19929_b200 as pkg
    import workloads as wl
    rng = np.random.default_rng(21)
    tags = wl.tags_with_spans(rng, T, 300)
    c_t, c_v = wl.outlier_sets(rng, D_IN, 16)
    x = wl.make_activations(rng, T, D_IN, tags, c_t, c_v, dtype=np.float16)
    col_max = np.max(np.abs(x.astype(np.float64)), axis=0)
    layer = wl.build_split_layer(pkg, rng, wl.LayerSpec("dist", D_IN, D_OUT, 16, 16, 8, 12), col_max,
                                 c_t, c_v)
    return layer, x, tags


def _run_rows(layer, x, tags):
    from paper_2605_19929_b200 import runtime
    gl = runtime.packed(layer)
    xd = torch.from_numpy(x).cuda()
    td = torch.from_numpy(tags).cuda()
    raw = gl.run(xd, td, raw=True)
    y = gl.run(xd, td)
    torch.cuda.synchronize()
    return raw[0].cpu(), y.cpu()


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2605_19929_b200 import parallel
        layer, x, tags = _case()
        lo, hi = parallel.token_shard(T, rank, world)
        acc, y = _run_rows(layer, x[lo:hi], tags[lo:hi])
        acc_all = parallel.gather_rows(acc, T)
        y_all = parallel.gather_rows(y, T)
        q.put((rank, (acc_all.numpy(), y_all.numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_token_sharded_forward_gpu_kernels(world):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import splitq_oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    layer, x, tags = _case()
    acc1, _ = _run_rows(layer, x, tags)
    ref = orc.forward(orc.from_reference_layer(layer), x.astype(np.float64), tags)
    rms = np.sqrt(np.mean(ref ** 2))
    for r in range(world):
        acc, y = out[r]
        np.testing.assert_array_equal(acc, acc1.numpy())
        assert np.max(np.abs(y.astype(np.float64) - ref)) <= 1e-3 * rms
