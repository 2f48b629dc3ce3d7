"""GPU MOCD statistics vs the reference (golden fixtures) and the oracle:
vision scores and percentile ranks exact, text scores bit-identical,
partitions identical."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import mocd_oracle as mo

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _pkg():
    import paper_2605_19929_b200 as pkg
    from paper_2605_19929_b200 import mocd_gpu
    return pkg, mocd_gpu


def test_golden_mocd_cases():
    pkg, mg = _pkg()
    d = np.load(os.path.join(GOLD, "mocd.npz"))
    for pre in ("s0_", "s1_", "s2_", "r0_", "r1_", "r2_"):
        x, tags = d[pre + "x"], d[pre + "tags"]
        k = int(d[pre + "k"]) if pre + "k" in d else 3
        ratio = 2 / 64 if pre.startswith("s") else 0.125
        batch = pkg.ActivationBatch(x, tags)
        if pre + "vscore" in d:
            np.testing.assert_array_equal(mg.vision_score(batch), d[pre + "vscore"])
            cand = np.setdiff1d(np.arange(x.shape[1]), d[pre + "c_vision"])
            np.testing.assert_array_equal(mg.percentile_rank(batch, cand), d[pre + "ranks"])
        part = mg.build_partition(batch, pkg.MocdConfig(ratio, ratio, clusters_k=k))
        np.testing.assert_array_equal(part.c_text, d[pre + "c_text"])
        np.testing.assert_array_equal(part.c_vision, d[pre + "c_vision"])
        cand = np.setdiff1d(np.arange(x.shape[1]), part.c_vision)
        counts = mg._GPU.rank_counts(torch.from_numpy(x).cuda(), torch.from_numpy(tags).cuda(), cand)
        ts = mg.text_score_counts(counts, cand.size, min(k, int((tags == 0).sum()))).cpu().numpy()
        np.testing.assert_array_equal(ts, d[pre + "tscore"])


@pytest.mark.parametrize("seed,n_text,n_vis,dim,k,dtype", [
    (0, 300, 100, 96, 3, np.float32), (1, 1000, 200, 257, 3, np.float16),
    (2, 129, 40, 64, 2, np.float64), (3, 700, 100, 130, 4, np.float32),
    (4, 64, 64, 40, 1, np.float32), (5, 2000, 500, 512, 3, np.float16),
    # long member sequences: many pairwise leaves per cluster (parallel exact sums)
    (6, 30000, 1000, 24, 3, np.float16), (7, 20000, 100, 16, 1, np.float32),
    (9, 25000, 500, 20, 8, np.float32)])
def test_random_batches_bit_exact(seed, n_text, n_vis, dim, k, dtype):
    pkg, mg = _pkg()
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((n_text + n_vis, dim)) * rng.uniform(0.05, 8, dim)).astype(dtype)
    if seed % 2:  # exact ties and repeated values in the ranks
        x[:, ::7] = np.round(x[:, ::7])
    tags = rng.permutation(np.array([0] * n_text + [1] * n_vis, np.uint8))
    xd = x.astype(np.float64)
    np.testing.assert_array_equal(mg._GPU.absmax(torch.from_numpy(x).cuda(),
                                                 torch.from_numpy(tags).cuda())[0].cpu().numpy(),
                                  mo.vision_score(xd, tags))
    cand = np.arange(dim)[rng.random(dim) > 0.1]
    counts = mg._GPU.rank_counts(torch.from_numpy(x).cuda(), torch.from_numpy(tags).cuda(), cand)
    np.testing.assert_array_equal(counts.cpu().numpy().astype(np.int64) & 0xFFFF,
                                  mo.rank_counts(xd, tags, cand))
    ts = mg.text_score_counts(counts, cand.size, k).cpu().numpy()
    ref = mo.text_score(mo.percentile_rank(xd, tags, cand), k, 50)
    np.testing.assert_array_equal(ts, ref)
    cfg = pkg.MocdConfig(0.05, 0.05, clusters_k=k)
    part = mg.build_partition(pkg.ActivationBatch(xd, tags), cfg)
    c_main, c_text, c_vision = mo.build_partition(xd, tags, 0.05, 0.05, k)
    np.testing.assert_array_equal(part.c_text, c_text)
    np.testing.assert_array_equal(part.c_vision, c_vision)


def test_topk_ties_to_lower_index():
    _, mg = _pkg()
    s = torch.tensor([3.0, 1.0, 3.0, 2.0, 3.0], dtype=torch.float64, device="cuda")
    assert mg._GPU.topk(s, 2).cpu().tolist() == [0, 2]
    assert mg._GPU.topk(s, 4).cpu().tolist() == [0, 2, 3, 4]


def test_errors():
    pkg, mg = _pkg()
    b = pkg.ActivationBatch(np.ones((4, 8)), [0, 0, 0, 0])
    with pytest.raises(ValueError, match="vision"):
        mg.build_partition(b, pkg.MocdConfig(ratio_vision=0.25, ratio_text=0.0))
    with pytest.raises(ValueError, match="vision"):
        mg.vision_score(b)


def test_stability_report_matches_reference():
    """calibrate.stability_report on the device against the reference's own
    report (tests/golden/stability.npz, gen_golden.py gen_stability)."""
    import os
    pkg, _ = _pkg()
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "stability.npz"))
    cfg = pkg.MocdConfig(float(d["ratios"][0]), float(d["ratios"][1]))
    batch = pkg.ActivationBatch(torch.from_numpy(d["x"]).cuda(), torch.from_numpy(d["tags"]).cuda())
    rep = pkg.stability_report(batch, cfg, [int(s) for s in d["sizes"]], int(d["ref_size"]),
                               int(d["trials"]), seed=2)
    np.testing.assert_array_equal([r["mean_jaccard"] for r in rep], d["mean"])
    np.testing.assert_array_equal([r["std_jaccard"] for r in rep], d["std"])
    assert [r["subset_size"] for r in rep] == [int(s) for s in d["sizes"]]


@pytest.mark.parametrize("n_cand_dim", [40, 3000])
def test_rank_counts_bf16_histogram(n_cand_dim):
    """bf16 rows take the 16-bit histogram rank counts (as fp16 rows do);
    counts equal the oracle's on the exact values the bf16 rows hold."""
    _, mg = _pkg()
    rng = np.random.default_rng(11 + n_cand_dim)
    n_text, n_vis = 300, 50
    x = rng.standard_normal((n_text + n_vis, n_cand_dim)) * rng.uniform(0.05, 8, n_cand_dim)
    x[:, ::5] = np.round(x[:, ::5])  # repeated keys (ties count via <=)
    xt = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)
    xd = xt.float().numpy().astype(np.float64)
    tags = rng.permutation(np.array([0] * n_text + [1] * n_vis, np.uint8))
    cand = np.arange(n_cand_dim)[rng.random(n_cand_dim) > 0.1]
    counts = mg._GPU.rank_counts(xt.cuda(), torch.from_numpy(tags).cuda(), cand)
    np.testing.assert_array_equal(counts.cpu().numpy().astype(np.int64) & 0xFFFF,
                                  mo.rank_counts(xd, tags, cand))


@pytest.mark.parametrize("n_text,k", [(1001, 3), (77, 4), (3, 2)])
def test_text_score_unpadded_rows(n_text, k):
    """The C-ABI text score on a transposed count matrix whose row stride is
    not a whole number of 16-byte vectors (rows alternate between the vector
    and the scalar reader, and between the vectorised and the scalar
    compaction): scores equal the oracle's k-means bit for bit. The buffer
    extends one vector past the last row (the contract in splitq.h)."""
    import ctypes as C
    from paper_2605_19929_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(1000 + n_text)
    n_cand, w = 300, 37
    counts = rng.integers(1, n_cand + 1, (n_text, w))
    counts[:, ::5] = rng.integers(1, 4, (n_text, len(range(0, w, 5))))  # few levels
    ld = n_text  # no padding between rows
    buf = np.zeros(w * ld + 16, np.int16)
    buf[: w * ld] = counts.T.reshape(-1).astype(np.int16)
    dev = torch.from_numpy(buf).cuda()
    scores = torch.zeros(w, dtype=torch.float64, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.splitq_mocd_text_score(dev.data_ptr(), ld, n_cand, n_text, k, 50, 0, w,
                                          scores.data_ptr(), st))
    got = scores.cpu().numpy()
    ref = np.array([mo.kmeans_1d_exact(counts[:, c], n_cand, min(k, n_text), 50) for c in range(w)])
    np.testing.assert_array_equal(got, ref)
