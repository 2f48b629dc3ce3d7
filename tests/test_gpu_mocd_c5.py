"""MOCD statistics at BASELINE config-5 size (128 x 2048 tokens, 25 %
vision, D = 3584: 196,608 text rows) against the oracle (mocd.py:72-150) on
sampled channels: the vision score, the rank counts of every text row
(percentile_rank numerators) and the k-means text score of each sampled
channel are bit-exact; the partition is the stable top-k of the device
scores (mocd.py:153-179)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import mocd_oracle as mo

pytestmark = pytest.mark.gpu

SAMPLES, SEQ, D = 128, 2048, 3584


def test_c5_sampled_channels_bit_exact():
    import paper_2605_19929_b200 as pkg
    from paper_2605_19929_b200 import mocd_gpu as mg
    rng = np.random.default_rng(55)
    T = SAMPLES * SEQ
    tags = np.concatenate([rng.permutation(np.array([1] * (SEQ // 4) + [0] * (SEQ - SEQ // 4), np.uint8))
                           for _ in range(SAMPLES)])
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    x = torch.randn((T, D), generator=g, device="cuda", dtype=torch.float32)
    planted_v, planted_t = np.arange(10, 42), np.arange(100, 132)
    td = torch.from_numpy(tags).cuda()
    vis = (td == 1).unsqueeze(1)
    x[:, planted_v] = torch.where(vis, x[:, planted_v] * 40.0, x[:, planted_v])
    # text-instability: channels whose magnitude rank jumps between token groups
    jump = torch.from_numpy(rng.uniform(0.2, 6.0, (T, 1))).cuda().float()
    x[:, planted_t] = torch.where(~vis, x[:, planted_t] * jump, x[:, planted_t])
    x = x.to(torch.float16)

    vmax, _ = mg._GPU.absmax(x, td)
    cfg = pkg.MocdConfig()  # reference defaults: 2 % + 2 %, k = 3, 50 iterations
    c_vision = mg._GPU.topk(vmax, cfg.k_vision(D)).cpu().numpy()
    cand = np.setdiff1d(np.arange(D), c_vision)
    counts = mg._GPU.rank_counts(x, td, cand)
    scores = mg.text_score_counts(counts, cand.size, cfg.clusters_k).cpu().numpy()
    part = mg.build_partition(pkg.ActivationBatch(x, td), cfg)
    np.testing.assert_array_equal(part.c_vision, np.sort(c_vision))
    np.testing.assert_array_equal(part.c_text, cand[mo.select_topk(scores, cfg.k_text(D))])

    xh = x.cpu().numpy()
    text = tags == 0
    a_text = np.abs(xh[text][:, cand].astype(np.float32))  # fp16 -> fp32 is exact
    np.testing.assert_array_equal(vmax.cpu().numpy(), np.max(np.abs(xh[tags == 1]), axis=0).astype(np.float64))  # mocd.py:72-77
    cnt = counts.cpu().numpy().view(np.uint16)
    sample = np.concatenate([rng.choice(cand.size, 4, replace=False),
                             np.searchsorted(cand, np.intersect1d(cand, planted_t[:3]))])
    for j in sample:
        ref_counts = (a_text <= a_text[:, j:j + 1]).sum(axis=1)  # mocd.py:106-110 (side="right")
        np.testing.assert_array_equal(cnt[:, j].astype(np.int64), ref_counts)
        ref_score = mo.kmeans_1d(ref_counts / cand.size, cfg.clusters_k, cfg.kmeans_max_iter)
        assert scores[j] == ref_score, (j, scores[j], ref_score)
