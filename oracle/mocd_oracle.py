"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see splitq_oracle.py header).

numpy restatement of MOCD channel selection
(/root/reference/pkg/src/modquant/mocd.py), plus the histogram formulation
of the text score that the GPU statistics kernels implement:

  percentile_rank(i, c) = count(i, c) / |C'|, count = #{j in C' : |x_ij| <= |x_ic|}
  (mocd.py:92-111) takes only |C'| distinct values per channel, so a channel's
  rank sequence is fully described by the histogram h_c[v] = #{text rows with
  count v}; the 1-D k-means (mocd.py:114-138) is then run on (value, weight)
  pairs. The histograms are additive over token shards, which is what makes
  the multi-GPU reduction an NCCL SUM all-reduce.
"""

from __future__ import annotations

import numpy as np


def vision_score(x, tags):  # mocd.py:72-77
    rows = np.flatnonzero(np.asarray(tags) == 1)
    if rows.size == 0:
        raise ValueError("no vision tokens present")
    return np.max(np.abs(np.asarray(x, np.float64)[rows]), axis=0)


def column_absmax(x):  # transform.py:89 (init_transform statistic)
    return np.max(np.abs(np.asarray(x, np.float64)), axis=0)


def select_topk(scores, k):  # mocd.py:80-89
    scores = np.asarray(scores, dtype=np.float64)
    if k > scores.shape[0]:
        raise ValueError(f"k={k} exceeds score vector length {scores.shape[0]}")
    if k == 0:
        return np.empty(0, dtype=np.int64)
    order = np.argsort(-scores, kind="stable")
    return np.sort(order[:k]).astype(np.int64)


def rank_counts(x, tags, cand):
    """Integer numerators of percentile_rank (mocd.py:106-110)."""
    cand = np.asarray(cand, np.int64)
    rows = np.flatnonzero(np.asarray(tags) == 0)
    a = np.abs(np.asarray(x, np.float64)[np.ix_(rows, cand)])
    counts = np.empty(a.shape, np.int64)
    for i in range(a.shape[0]):
        srt = np.sort(a[i])
        counts[i] = np.searchsorted(srt, a[i], side="right")
    return counts


def percentile_rank(x, tags, cand):  # mocd.py:92-111
    cand = np.asarray(cand, np.int64)
    if cand.size == 0:
        raise ValueError("candidate channel set is empty")
    return rank_counts(x, tags, cand) / cand.size


def kmeans_1d(values, k, max_iter):  # mocd.py:114-138
    values = np.asarray(values, np.float64)
    distinct = np.unique(values)
    k = min(k, distinct.size)
    if k == 1:
        return float(np.var(values))
    quantiles = (2 * np.arange(1, k + 1) - 1) / (2 * k)
    centers = np.quantile(values, quantiles)
    assign = np.argmin(np.abs(values[:, None] - centers[None, :]), axis=1)
    for _ in range(max_iter):
        new_centers = centers.copy()
        for j in range(k):
            members = values[assign == j]
            if members.size:
                new_centers[j] = members.mean()
        new_assign = np.argmin(np.abs(values[:, None] - new_centers[None, :]), axis=1)
        centers = new_centers
        if np.array_equal(new_assign, assign):
            break
        assign = new_assign
    return float(np.mean((values - centers[assign]) ** 2))


def text_score(ranks, k, max_iter=50):  # mocd.py:141-150
    if k < 1:
        raise ValueError("cluster count must be positive")
    if k > ranks.shape[0]:
        raise ValueError("cluster count exceeds number of text tokens")
    return np.array([kmeans_1d(ranks[:, c], k, max_iter) for c in range(ranks.shape[1])])


def build_partition(x, tags, ratio_vision=0.02, ratio_text=0.02, clusters_k=3,
                    kmeans_max_iter=50):  # mocd.py:153-179
    x = np.asarray(x, np.float64)
    tags = np.asarray(tags)
    dim = x.shape[1]
    k_v = int(np.floor(ratio_vision * dim + 0.5))
    k_t = int(np.floor(ratio_text * dim + 0.5))
    all_c = np.arange(dim)
    if k_v > 0:
        if not np.any(tags == 1):
            raise ValueError("nonzero vision ratio but no vision tokens")
        c_vision = select_topk(vision_score(x, tags), k_v)
    else:
        c_vision = np.empty(0, np.int64)
    remaining = np.setdiff1d(all_c, c_vision)
    if k_t > 0:
        n_text = int(np.sum(tags == 0))
        if n_text == 0:
            raise ValueError("nonzero text ratio but no text tokens")
        ranks = percentile_rank(x, tags, remaining)
        scores = text_score(ranks, min(clusters_k, ranks.shape[0]), kmeans_max_iter)
        c_text = remaining[select_topk(scores, k_t)]
    else:
        c_text = np.empty(0, np.int64)
    c_main = np.setdiff1d(all_c, np.concatenate([c_vision, c_text]))
    return c_main, c_text, c_vision


# ---------------------------------------------------------------- histogram form

def rank_histograms(counts, n_cand):
    """h[c, v] = #{text rows whose count for channel c is v}, v in 0..n_cand."""
    counts = np.asarray(counts, np.int64)
    h = np.zeros((counts.shape[1], n_cand + 1), np.int64)
    for c in range(counts.shape[1]):
        h[c] = np.bincount(counts[:, c], minlength=n_cand + 1)
    return h


def kmeans_1d_hist(hist, n_cand, k, max_iter):
    """mocd.py:114-138 on the (value = v / n_cand, weight = hist[v]) form.

    Same initialisation (np.quantile linear interpolation at (n - 1) q on the
    sorted multiset), same assignment rule (nearest centre, ties to the lower
    index), same empty-cluster rule and stopping test; centre means are
    computed as exact integer sums divided once, so they may differ from the
    reference's pairwise fp64 mean by an ulp."""
    hist = np.asarray(hist, np.int64)
    levels = np.flatnonzero(hist)
    vals = levels / n_cand
    w = hist[levels]
    n = int(w.sum())
    k = min(k, levels.size)
    if k == 1:
        mean = (levels * w).sum() / n_cand / n
        return float(((vals - mean) ** 2 * w).sum() / n)
    cum = np.cumsum(w)

    def order_stat(idx):  # value of the idx-th element (0-based) of the sorted multiset
        return vals[np.searchsorted(cum, idx, side="right")]

    centers = np.empty(k)
    qs = (2 * np.arange(1, k + 1) - 1) / (2 * k)
    for j in range(k):
        # numpy 'linear' quantile (numpy/lib/_function_base_impl.py): virtual
        # index (n - 1) * q, neighbours clamped to the last element, lerp that
        # switches to b - (b - a)(1 - t) for t >= 0.5
        vi = (n - 1) * qs[j]
        if vi >= n - 1:
            lo = hi = n - 1
        else:
            lo = int(np.floor(vi))
            hi = lo + 1
        t = vi - np.floor(vi)
        a = order_stat(lo)
        b = order_stat(hi)
        diff = b - a
        centers[j] = b - diff * (1 - t) if t >= 0.5 else a + diff * t
    assign = np.argmin(np.abs(vals[:, None] - centers[None, :]), axis=1)
    for _ in range(max_iter):
        new_centers = centers.copy()
        for j in range(k):
            m = assign == j
            cnt = w[m].sum()
            if cnt:
                new_centers[j] = (levels[m] * w[m]).sum() / n_cand / cnt
        new_assign = np.argmin(np.abs(vals[:, None] - new_centers[None, :]), axis=1)
        centers = new_centers
        if np.array_equal(new_assign, assign):
            break
        assign = new_assign
    return float((((vals - centers[assign]) ** 2) * w).sum() / n)


def text_score_hist(hists, n_cand, k, max_iter=50):
    return np.array([kmeans_1d_hist(h, n_cand, k, max_iter) for h in hists])


# ---------------------------------------------------------------- exact streaming form

def pairwise_sum(a):
    """numpy's float64 add.reduce: 8-accumulator pairwise summation
    (numpy/_core/src/umath/loops_utils.h.src pairwise_sum), verified
    bit-for-bit against np.sum in tests/test_oracle_golden.py."""
    def pw(lo, n):
        if n < 8:
            res = 0.0
            for i in range(n):
                res += a[lo + i]
            return res
        if n <= 128:
            r = [a[lo + j] for j in range(8)]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return pw(lo, n2) + pw(lo + n2, n - n2)
    a = [float(v) for v in a]
    return pw(0, len(a))


def kmeans_1d_exact(counts, n_cand, k, max_iter):
    """_kmeans_1d (mocd.py:114-138) on one channel's rank counts in token
    order, written the way the GPU kernel evaluates it: values v = c / n_cand,
    order statistics from a counting sort, per-level assignment, centre means
    as numpy pairwise sums over the members in token order. Bit-identical to
    the reference (checked in tests)."""
    counts = np.asarray(counts, np.int64)
    vals = counts / n_cand
    n = vals.size
    hist = np.bincount(counts, minlength=n_cand + 1)
    levels = np.flatnonzero(hist)
    k = min(k, levels.size)
    if k == 1:
        mean = pairwise_sum(vals) / n
        dev = vals - mean
        return pairwise_sum(dev * dev) / n
    cum = np.cumsum(hist)

    def order_stat(idx):
        return np.searchsorted(cum, idx, side="right") / n_cand

    qs = (2 * np.arange(1, k + 1) - 1) / (2 * k)
    centers = np.empty(k)
    for j in range(k):
        vi = (n - 1) * qs[j]
        lo = int(np.floor(vi)) if vi < n - 1 else n - 1
        hi = lo + 1 if vi < n - 1 else n - 1
        t = vi - np.floor(vi)
        a, b = order_stat(lo), order_stat(hi)
        diff = b - a
        centers[j] = b - diff * (1 - t) if t >= 0.5 else a + diff * t

    def assign_levels(c):
        lv = levels / n_cand
        return np.argmin(np.abs(lv[:, None] - c[None, :]), axis=1)

    lvl_of = np.full(n_cand + 1, -1, np.int64)
    lvl_of[levels] = np.arange(levels.size)
    assign = assign_levels(centers)
    for _ in range(max_iter):
        new_centers = centers.copy()
        a_tok = assign[lvl_of[counts]]
        for j in range(k):
            members = vals[a_tok == j]
            if members.size:
                new_centers[j] = pairwise_sum(members) / members.size
        new_assign = assign_levels(new_centers)
        centers = new_centers
        if np.array_equal(new_assign, assign):
            break
        assign = new_assign
    dev = vals - centers[assign[lvl_of[counts]]]
    return pairwise_sum(dev * dev) / n


class PairwiseStream:
    """numpy's pairwise summation of a stream of known length n, consuming
    one value at a time (post-order evaluation of the recursion tree:
    segments > 128 split at n2 = n/2 - (n/2) % 8, leaves of >= 8 elements use
    8 accumulators, leaves of < 8 a sequential sum from 0.0). This is the
    exact algorithm of the GPU text-score kernel (csrc/mocd.cu)."""

    def __init__(self, n):
        self.stack = []  # frames [seg_len, n2, phase, left_sum]
        self.total = None
        if n == 0:
            self.total = 0.0
            return
        self._descend(n)

    def _descend(self, m):
        while m > 128:
            n2 = m // 2
            n2 -= n2 % 8
            self.stack.append([m, n2, 0, 0.0])
            m = n2
        self.leaf_len, self.leaf_i = m, 0
        self.r = [0.0] * 8
        self.res = 0.0

    def push(self, v):
        m, i = self.leaf_len, self.leaf_i
        if m < 8:
            self.res += v
        else:
            body = m - m % 8
            if i < 8:
                self.r[i] = v
            elif i < body:
                self.r[i % 8] += v
            else:
                if i == body:
                    r = self.r
                    self.res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
                self.res += v
            if i == m - 1 and body == m:
                r = self.r
                self.res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        self.leaf_i = i + 1
        if self.leaf_i == m:
            self._finish_leaf(self.res)

    def _finish_leaf(self, s):
        while self.stack:
            f = self.stack[-1]
            if f[2] == 0:
                f[2], f[3] = 1, s
                self._descend(f[0] - f[1])
                return
            s = f[3] + s
            self.stack.pop()
        self.total = s
