"""A reference-written layer directory straight to the device (SURVEY 8(f)
row 2): load_layer_packed packs once, caches the blob next to the manifest
and reuses it; outputs match the reference's forward on the fixture batch
(tests/golden/layer_dir, written by modquant.save_layer / save_tensor)."""
import os
import shutil

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_19929_b200 as pkg
from paper_2605_19929_b200 import layer_io, runtime

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "layer_dir")


def _run(gl, batch, raw=False):
    x = torch.from_numpy(np.ascontiguousarray(batch.data)).cuda()
    t = torch.from_numpy(batch.tags).cuda()
    y = gl.run(x, t, raw=raw)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def test_load_layer_packed_matches_reference(tmp_path):
    d = tmp_path / "layer"
    shutil.copytree(GOLD, d)
    man = str(d / "manifest.json")
    batch = pkg.load_tensor(str(d / "batch.spqt"))
    y_ref = np.load(str(d / "y_ref.npy"))
    g1 = pkg.load_layer_packed(man)
    blob = d / layer_io.PACKED_NAME
    assert blob.exists()
    stamp = blob.stat().st_mtime_ns
    g2 = pkg.load_layer_packed(man)  # from the cached blob
    assert blob.stat().st_mtime_ns == stamp
    g3 = runtime.GpuLayer(pkg.load_layer(man))  # packed afresh
    r1, r2, r3 = (_run(g, batch, raw=True) for g in (g1, g2, g3))
    np.testing.assert_array_equal(r1[0], r3[0])  # int32 main accumulators
    np.testing.assert_array_equal(r1, r2)
    y = _run(g2, batch).astype(np.float64)
    rms = np.sqrt(np.mean(y_ref ** 2))
    assert np.max(np.abs(y - y_ref)) <= 1e-3 * rms
    # a changed tensor invalidates the blob
    w = pkg.load_tensor(str(d / "w_vision.spqt"))
    pkg.save_tensor(str(d / "w_vision.spqt"), w * 2.0)
    pkg.load_layer_packed(man)
    assert blob.stat().st_mtime_ns != stamp
