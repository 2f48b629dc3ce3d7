"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 path.

The forward shards tokens by rows with no collective on the path
(per-token quantization, row-local MAC); gathering the shards must give the
single-process result bit for bit. The CPU oracle stands in for the device
kernels here (test infrastructure), the sharding and collectives are the
product's (paper_2605_19929_b200.parallel).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


def _case():
    import paper_2605_19929_b200 as pkg
    import workloads as wl
    rng = np.random.default_rng(3)
    T, d_in, d_out = 96, 128, 64
    tags = wl.tags_with_spans(rng, T, 24)
    c_t, c_v = wl.outlier_sets(rng, d_in, 4)
    x = wl.make_activations(rng, T, d_in, tags, c_t, c_v, dtype=np.float32).astype(np.float64)
    col_max = np.max(np.abs(x), axis=0)
    layer = wl.build_split_layer(pkg, rng, wl.LayerSpec("t", d_in, d_out, 4, 4, 4, 6), col_max,
                                 c_t, c_v)
    return layer, x, tags


def _sharded_forward(rank, world):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import splitq_oracle as orc
    from paper_2605_19929_b200 import parallel
    layer, x, tags = _case()
    lo, hi = parallel.token_shard(x.shape[0], rank, world)
    y_local = orc.forward(orc.from_reference_layer(layer), x[lo:hi], tags[lo:hi])
    y = parallel.gather_rows(torch.from_numpy(y_local), x.shape[0])
    return y.numpy()


def test_token_sharded_forward_equals_single_process():
    from oracle import splitq_oracle as orc
    outs = spawn(_sharded_forward)
    layer, x, tags = _case()
    ref = orc.forward(orc.from_reference_layer(layer), x, tags)
    for y in outs:
        np.testing.assert_array_equal(y, ref)


def test_token_shard_partition_covers_rows():
    from paper_2605_19929_b200 import parallel
    for T in (1, 7, 64, 65536, 65537):
        for world in (1, 2, 4, 8):
            spans = [parallel.token_shard(T, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == T
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
