"""The distributed MOCD path (mocd_gpu.build_partition_distributed,
mocd.py:153-179 over token shards) with the product's sm_100a statistics
kernels on every rank: world_size 2 and 3 on one GPU, the collectives over
gloo on host copies of the per-shard results (the ranks' kernels never wait
on one another). The partition must equal the single-process reference's.
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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(seed, n_text, n_vis, dim):
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((n_text + n_vis, dim)) * rng.uniform(0.05, 8, dim)).astype(np.float16)
    tags = rng.permutation(np.array([0] * n_text + [1] * n_vis, np.uint8))
    return x, tags


def _worker(rank, world, port, args, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2605_19929_b200 import mocd_gpu, parallel
        from paper_2605_19929_b200.mocd import MocdConfig

        class HostCollStats(mocd_gpu.GpuStats):
            """The GPU kernels, results handed to the collectives on the host."""

            def absmax(self, x, tags):
                v, a = super().absmax(x, tags)
                return v.cpu(), a.cpu()

            def rank_counts(self, x, tags, cand):
                return super().rank_counts(x, tags, cand).cpu()

            def text_score(self, counts, n_cand, k, max_iter):
                return super().text_score(counts.cuda(), n_cand, k, max_iter).cpu()

            def topk(self, scores, k):
                return super().topk(scores.cuda(), k).cpu()

        seed, n_text, n_vis, dim, k = args
        x, tags = _case(seed, n_text, n_vis, dim)
        lo, hi = parallel.token_shard(x.shape[0], rank, world)
        xd = torch.from_numpy(x[lo:hi]).cuda()
        td = torch.from_numpy(tags[lo:hi]).cuda()
        p = mocd_gpu.build_partition_distributed(xd, td, MocdConfig(0.05, 0.05, clusters_k=k),
                                                 stats=HostCollStats())
        q.put((rank, (p.c_main, p.c_text, p.c_vision)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,args", [(2, (0, 1500, 500, 300, 3)), (3, (1, 2000, 300, 257, 4))])
def test_distributed_partition_gpu_kernels_equal_reference(world, args):
    from oracle import mocd_oracle as mo
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    seed, n_text, n_vis, dim, k = args
    x, tags = _case(seed, n_text, n_vis, dim)
    ref = mo.build_partition(x.astype(np.float64), tags, 0.05, 0.05, k)
    for r in range(world):
        for a, b in zip(out[r], ref):
            np.testing.assert_array_equal(a, b)
