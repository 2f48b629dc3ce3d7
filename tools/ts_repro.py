#!/usr/bin/env python
"""Text-score kernel at C5 token counts against the oracle (debug aid)."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_19929_b200 import mocd_gpu as mg  # noqa: E402
from oracle import mocd_oracle as mo  # noqa: E402

n_text, n_cand, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(0)
counts = torch.from_numpy(rng.integers(1, n_cand + 1, (n_text, n_cand)).astype(np.int16)).cuda()
ts = mg.text_score_counts(counts, n_cand, k).cpu().numpy()
torch.cuda.synchronize()
if len(sys.argv) > 4:
    c = counts.cpu().numpy().astype(np.int64)
    ref = np.array([mo.kmeans_1d(c[:, j] / n_cand, k, 50) for j in range(min(n_cand, 8))])
    print("max diff", np.max(np.abs(ts[:len(ref)] - ref)), "equal", np.array_equal(ts[:len(ref)], ref))
print("ok", ts[:4])
