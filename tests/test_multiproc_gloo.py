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
    out = dict(q.get(timeout=120) for _ in procs)
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


class OracleStats:
    """CPU stand-in for the per-shard GPU statistics (test infrastructure)."""

    def absmax(self, x, tags):
        from oracle import mocd_oracle as mo
        x = np.asarray(x, np.float64)
        tags = np.asarray(tags)
        v = np.max(np.abs(x[tags == 1]), axis=0) if np.any(tags == 1) else np.zeros(x.shape[1])
        return torch.from_numpy(v), torch.from_numpy(mo.column_absmax(x))

    def rank_counts(self, x, tags, cand):
        from oracle import mocd_oracle as mo
        return torch.from_numpy(mo.rank_counts(x, tags, cand).astype(np.int16))

    def text_score(self, counts, n_cand, k, max_iter):
        from oracle import mocd_oracle as mo
        cnt = counts.numpy().astype(np.int64) & 0xFFFF
        return torch.from_numpy(np.array([mo.kmeans_1d_exact(cnt[:, c], n_cand, k, max_iter)
                                          for c in range(cnt.shape[1])]))

    def topk(self, scores, k):
        from oracle import mocd_oracle as mo
        return torch.from_numpy(mo.select_topk(scores.numpy(), k))


def _mocd_case():
    rng = np.random.default_rng(11)
    n, dim = 90, 40
    x = rng.standard_normal((n, dim)) * rng.uniform(0.1, 4, dim)
    x[:, 3] *= 30
    tags = rng.permutation(np.array([0] * 60 + [1] * 30, np.uint8))
    x[tags == 1, 7] *= 50
    return x, tags


def _sharded_partition(rank, world):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2605_19929_b200 import mocd_gpu, parallel
    from paper_2605_19929_b200.mocd import MocdConfig
    x, tags = _mocd_case()
    lo, hi = parallel.token_shard(x.shape[0], rank, world)
    p = mocd_gpu.build_partition_distributed(x[lo:hi], tags[lo:hi],
                                             MocdConfig(0.1, 0.1, clusters_k=3),
                                             stats=OracleStats())
    return p.c_main, p.c_text, p.c_vision


def test_mocd_partition_distributed_equals_single_process():
    from oracle import mocd_oracle as mo
    x, tags = _mocd_case()
    ref = mo.build_partition(x, tags, 0.1, 0.1, 3)
    for out in spawn(_sharded_partition):
        for a, b in zip(out, ref):
            np.testing.assert_array_equal(a, b)


def _exchange(rank, world):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2605_19929_b200 import mocd_gpu
    full = torch.arange(23 * 10, dtype=torch.int16).view(23, 10)
    bounds = [r * 23 // world for r in range(world + 1)]  # uneven row shards
    got, c0, c1 = mocd_gpu._exchange_columns(full[bounds[rank]:bounds[rank + 1]].clone(), 10, world, rank, None)
    return got.numpy(), c0, c1


def test_rank_count_column_exchange_world3():
    """The all-to-all gives each rank its channel range of every row, in
    token order (uneven row and column splits)."""
    full = np.arange(23 * 10, dtype=np.int16).reshape(23, 10)
    for got, c0, c1 in spawn(_exchange, world=3):
        np.testing.assert_array_equal(got, full[:, c0:c1])


def test_mocd_partition_distributed_world3():
    from oracle import mocd_oracle as mo
    x, tags = _mocd_case()
    ref = mo.build_partition(x, tags, 0.1, 0.1, 3)
    for out in spawn(_sharded_partition, world=3):
        for a, b in zip(out, ref):
            np.testing.assert_array_equal(a, b)
