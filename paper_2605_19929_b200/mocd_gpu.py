"""MOCD calibration statistics on the GPU (reference: pkg/src/modquant/mocd.py).

Same names and semantics as the reference's vision_score / percentile_rank /
text_score / select_topk / build_partition, computed by the sm_100a kernels
in csrc/mocd.cu through the C-ABI. Scores are bit-identical to the
reference's numpy arithmetic (exact quantile init and pairwise-sum means), so
partitions are identical.

Token-sharded multi-GPU calibration (build_partition_distributed): each rank
reduces its own rows; per-channel absmax statistics are MAX-all-reduced, the
integer rank counts (percentile_rank numerators) are all-gathered in token
order, channels are sharded across ranks for the k-means text score, and the
scores are all-gathered; TopK then runs identically on every rank.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .mocd import ChannelPartition, MocdConfig, select_topk  # noqa: F401  (re-export)
from .tensor import _is_torch


def _torch():
    import torch

    return torch


def _stream():
    return C.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _dev_batch(x, tags):
    torch = _torch()
    from .runtime import device

    dev = device()
    if _is_torch(x):
        xt = x.to(dev)
    else:
        xt = torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.float64))).to(dev)
    if xt.stride(1) != 1:
        xt = xt.contiguous()
    tt = tags.to(dev) if _is_torch(tags) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(tags, np.uint8))).to(dev)
    return xt, tt.to(torch.uint8)


def _dt(t):
    from .runtime import _dtype_code

    return _dtype_code(t.dtype)


class GpuStats:
    """Per-shard statistics on the local GPU (the product backend)."""

    def absmax(self, x, tags):
        """(vision max |x|, all-rows max |x|) per channel, fp64 device tensors."""
        torch = _torch()
        lib = _lib.load()
        xt, tt = _dev_batch(x, tags)
        T, D = xt.shape
        vmax = torch.empty(D, dtype=torch.float64, device=xt.device)
        amax = torch.empty(D, dtype=torch.float64, device=xt.device)
        st = torch.zeros(4, dtype=torch.int32, device=xt.device)
        _lib.check(lib.splitq_mocd_absmax(xt.data_ptr(), _dt(xt), xt.stride(0), tt.data_ptr(), T, D,
                                          vmax.data_ptr(), amax.data_ptr(), st.data_ptr(), _stream()))
        s = C.c_int32()
        _lib.check(lib.splitq_read_status(C.c_void_p(st.data_ptr()), _stream(), C.byref(s)))
        return vmax, amax

    def rank_counts(self, x, tags, cand):
        """uint16 [n_text x n_cand] percentile_rank numerators (token order)."""
        torch = _torch()
        lib = _lib.load()
        xt, tt = _dev_batch(x, tags)
        rows = (tt == 0).nonzero().flatten().to(torch.int32)
        n_text = rows.numel()
        cand_t = torch.as_tensor(np.asarray(cand, np.int32), device=xt.device)
        counts = torch.empty((max(n_text, 1), cand_t.numel()), dtype=torch.int16, device=xt.device)
        if n_text == 0:
            return counts[:0]
        nt = torch.tensor([n_text], dtype=torch.int32, device=xt.device)
        _lib.check(lib.splitq_mocd_rank_counts(xt.data_ptr(), _dt(xt), xt.stride(0),
                                               rows.data_ptr(), nt.data_ptr(), n_text,
                                               cand_t.data_ptr(), cand_t.numel(),
                                               counts.data_ptr(), _stream()))
        return counts

    def text_score(self, counts, n_cand, k, max_iter):
        """fp64 [w]: _kmeans_1d of each of the w columns of ``counts``
        [n_text x w] (a column range of the percentile_rank numerators over
        n_cand candidates: n_cand is the ranks' denominator)."""
        torch = _torch()
        lib = _lib.load()
        n_text, w = int(counts.shape[0]), int(counts.shape[1])
        # rows padded to 8 tokens: the kernel reads them as 16-byte vectors
        counts_t = torch.empty((w, max((n_text + 7) // 8 * 8, 8)), dtype=torch.int16,
                               device=counts.device)
        if not counts.is_contiguous():
            counts = counts.contiguous()
        _lib.check(lib.splitq_mocd_transpose_u16(counts.data_ptr(), n_text, w,
                                                 counts_t.data_ptr(), counts_t.stride(0), _stream()))
        scores = torch.zeros(w, dtype=torch.float64, device=counts.device)
        _lib.check(lib.splitq_mocd_text_score(counts_t.data_ptr(), counts_t.stride(0), int(n_cand),
                                              n_text, int(k), int(max_iter), 0, w,
                                              scores.data_ptr(), _stream()))
        return scores

    def topk(self, scores, k):
        torch = _torch()
        lib = _lib.load()
        n = scores.numel()
        if k > n:
            raise ValueError(f"k={k} exceeds score vector length {n}")
        flags = torch.empty(max(n, 1), dtype=torch.int32, device=scores.device)
        out = torch.empty(max(k, 1), dtype=torch.int64, device=scores.device)
        if k == 0:
            return out[:0]
        _lib.check(lib.splitq_mocd_topk(scores.contiguous().data_ptr(), n, k, flags.data_ptr(),
                                        out.data_ptr(), _stream()))
        return out


_GPU = GpuStats()


# ---------------------------------------------------------------- reference API

def vision_score(batch):
    """mocd.py:72-77 (numpy result for numpy batches)."""
    tags = batch.tags.cpu().numpy() if _is_torch(batch.tags) else np.asarray(batch.tags)
    if not np.any(tags == 1):
        raise ValueError("no vision tokens present")
    vmax, _ = _GPU.absmax(batch.data, batch.tags)
    return vmax if _is_torch(batch.data) else vmax.cpu().numpy()


def channel_absmax(batch):
    """Per-channel max |x| over all rows: the init_transform statistic
    (transform.py:89) that build_layer(..., col_max=) consumes."""
    _, amax = _GPU.absmax(batch.data, batch.tags)
    return amax if _is_torch(batch.data) else amax.cpu().numpy()


def percentile_rank(batch, candidate_channels):
    """mocd.py:92-111."""
    cand = np.asarray(candidate_channels, dtype=np.int64)
    if cand.size == 0:
        raise ValueError("candidate channel set is empty")
    counts = _GPU.rank_counts(batch.data, batch.tags, cand)
    if counts.shape[0] == 0:
        raise ValueError("no text tokens present")
    # ranks / |C'| as an IEEE division (torch's CUDA tensor / scalar multiplies
    # by the reciprocal, which is not the reference's rounding)
    r = (counts.to(_torch().int32).cpu().numpy() & 0xFFFF) / cand.size
    return _torch().from_numpy(r).to(batch.data.device) if _is_torch(batch.data) else r


def text_score_counts(counts, n_cand, k, max_iter=50):
    """text_score (mocd.py:141-150) from the integer rank counts."""
    if k < 1:
        raise ValueError("cluster count must be positive")
    if k > counts.shape[0]:
        raise ValueError("cluster count exceeds number of text tokens")
    return _GPU.text_score(counts, n_cand, k, max_iter)


def text_score(ranks, k, max_iter=50):
    """text_score (mocd.py:141-150) with the reference's signature. The
    device k-means runs on integer rank counts, so ``ranks`` must be
    percentile_rank output: every entry an IEEE quotient count / n_cand with
    n_cand = ranks.shape[1] (checked exactly; anything else raises)."""
    torch = _torch()
    on_dev = _is_torch(ranks)
    r = ranks.detach().cpu().numpy() if on_dev else np.asarray(ranks, np.float64)
    if r.ndim != 2:
        raise ValueError(f"matrix must be 2-D, got ndim={r.ndim}")
    n_cand = int(r.shape[1])
    counts = np.rint(r * n_cand)
    if n_cand == 0 or n_cand > 65535 or not np.array_equal(counts / n_cand, r) or np.any(counts < 1):
        raise ValueError("text_score on the GPU takes percentile_rank output (counts / n_cand)")
    from .runtime import device

    c = torch.from_numpy(counts.astype(np.uint16).view(np.int16)).to(device())
    out = text_score_counts(c, n_cand, k, max_iter)
    return out if on_dev else out.cpu().numpy()


def build_partition(batch, cfg: MocdConfig) -> ChannelPartition:
    """mocd.py:153-179 on the GPU (this process's batch, no collectives)."""
    return build_partition_distributed(batch.data, batch.tags, cfg, group=False)


def build_partition_distributed(x_local, tags_local, cfg: MocdConfig, group=None,
                                stats=None) -> ChannelPartition:
    """build_partition over token shards (one per rank, rows in rank order;
    group=False: this process only).

    Collectives (torch.distributed, NCCL on GPUs): MAX all-reduce of the
    per-channel absmax, all-gather of the rank counts and of the channel-
    sharded scores. With no process group this is the single-GPU path.
    ``stats`` injects the per-shard statistics backend (default: the GPU
    kernels)."""
    torch = _torch()
    import torch.distributed as dist

    stats = stats or _GPU
    if group is False:  # explicit single-process call
        distributed, group = False, None
    else:
        distributed = dist.is_available() and dist.is_initialized() and \
            dist.get_world_size(group) > 1
    world = dist.get_world_size(group) if distributed else 1
    rank = dist.get_rank(group) if distributed else 0

    tags_np = tags_local.cpu().numpy() if _is_torch(tags_local) else np.asarray(tags_local, np.uint8)
    dim = int(x_local.shape[1])
    k_v, k_t = cfg.k_vision(dim), cfg.k_text(dim)

    def all_flag(v):
        t = torch.tensor([int(v)], dtype=torch.int64, device=_coll_device(stats))
        if distributed:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return bool(t.item())

    vmax, _ = stats.absmax(x_local, tags_local)
    if distributed:
        dist.all_reduce(vmax, op=dist.ReduceOp.MAX, group=group)
    if k_v > 0:
        if not all_flag(np.any(tags_np == 1)):
            raise ValueError("nonzero vision ratio but no vision tokens")
        c_vision = np.asarray(_to_np(stats.topk(vmax, k_v)), np.int64)
    else:
        c_vision = np.empty(0, np.int64)
    remaining = np.setdiff1d(np.arange(dim), c_vision)
    if k_t > 0:
        if not all_flag(np.any(tags_np == 0)):
            raise ValueError("nonzero text ratio but no text tokens")
        counts = stats.rank_counts(x_local, tags_local, remaining)
        n_cand = remaining.size
        if distributed:
            # channel-sharded k-means: every rank receives, for its own channel
            # range, the counts of all text rows in token (= rank) order
            counts, c0, c1 = _exchange_columns(counts, n_cand, world, rank, group)
        else:
            c0, c1 = 0, n_cand
        n_text = int(counts.shape[0])
        k = min(cfg.clusters_k, n_text)
        part = stats.text_score(counts, n_cand, k, cfg.kmeans_max_iter)
        scores = torch.zeros(n_cand, dtype=torch.float64, device=part.device)
        scores[c0:c1] = part
        if distributed:  # each rank filled its channel range, the rest is zero
            dist.all_reduce(scores, op=dist.ReduceOp.SUM, group=group)
        c_text = remaining[np.asarray(_to_np(stats.topk(scores, k_t)), np.int64)]
    else:
        c_text = np.empty(0, np.int64)
    c_main = np.setdiff1d(np.arange(dim), np.concatenate([c_vision, c_text]))
    return ChannelPartition(c_main, c_text, c_vision, dim)


def _to_np(t):
    return t.cpu().numpy() if _is_torch(t) else np.asarray(t)


def _coll_device(stats):
    torch = _torch()
    return torch.device("cuda", torch.cuda.current_device()) if stats is _GPU else torch.device("cpu")


def _exchange_columns(local, n_cand, world, rank, group):
    """All-to-all of the rank-count matrix: rank q gets columns
    [q n / W, (q + 1) n / W) of every rank's rows, stacked in rank (= token)
    order. Each rank receives n_text x n / W counts instead of the whole
    n_text x n matrix an all-gather would land on it (7.4 GB per
    rank at D = 18944)."""
    torch = _torch()
    import torch.distributed as dist

    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    rows = [int(v.item()) for v in sizes]
    bounds = [q * n_cand // world for q in range(world + 1)]
    c0, c1 = bounds[rank], bounds[rank + 1]
    esz = local.element_size()
    # NCCL / gloo have no 16-bit integer collectives: move the raw bytes
    send = torch.cat([local[:, bounds[q]:bounds[q + 1]].contiguous().reshape(-1).view(torch.uint8)
                      for q in range(world)])
    in_splits = [local.shape[0] * (bounds[q + 1] - bounds[q]) * esz for q in range(world)]
    out_splits = [r * (c1 - c0) * esz for r in rows]
    recv = torch.empty(sum(out_splits), dtype=torch.uint8, device=local.device)
    dist.all_to_all_single(recv, send, out_splits, in_splits, group=group)
    blocks, off = [], 0
    for r, b in zip(rows, out_splits):
        blocks.append(recv[off:off + b].view(local.dtype).view(r, c1 - c0))
        off += b
    return torch.cat(blocks, dim=0), c0, c1


def _gather_rows(local, world, group):
    """All-gather variable-length row blocks in rank (= token) order."""
    torch = _torch()
    import torch.distributed as dist

    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    width = max(sizes)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    # NCCL / gloo have no 16-bit integer collectives: move the raw bytes
    wire = pad.view(torch.uint8) if pad.dtype == torch.int16 else pad
    bufs = [torch.empty_like(wire) for _ in range(world)]
    dist.all_gather(bufs, wire, group=group)
    bufs = [b.view(pad.dtype) for b in bufs]
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)
