"""Layer state on disk: the reference's SPQT dumps and
layer directories read / written byte-identically, and the packed blob.

Fixture: tests/golden/layer_dir, written by the reference's own save_layer /
save_tensor (tests/golden/gen_golden.py gen_layer_dir).
"""
import filecmp
import json
import os
import shutil

import numpy as np
import pytest

import paper_2605_19929_b200 as pkg
from paper_2605_19929_b200 import layer_io, runtime

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "layer_dir")
MAN = os.path.join(GOLD, "manifest.json")


def test_spqt_round_trip_byte_identical(tmp_path):
    for name in ("matrix.spqt", "batch.spqt", "w_main.spqt", "p_main_scale.spqt"):
        obj = pkg.load_tensor(os.path.join(GOLD, name))
        out = tmp_path / name
        pkg.save_tensor(str(out), obj)
        assert filecmp.cmp(out, os.path.join(GOLD, name), shallow=False), name
    b = pkg.load_tensor(os.path.join(GOLD, "batch.spqt"))
    assert isinstance(b, pkg.ActivationBatch) and b.tags.dtype == np.uint8
    assert b.data.shape == (40, 48)


def _corrupt(tmp_path, raw, name="bad.spqt"):
    p = tmp_path / name
    p.write_bytes(raw)
    return str(p)


def test_spqt_errors(tmp_path):
    good = open(os.path.join(GOLD, "matrix.spqt"), "rb").read()
    batch = open(os.path.join(GOLD, "batch.spqt"), "rb").read()
    cases = {
        "truncated header": good[:10],
        "bad magic": b"XPQT" + good[4:],
        "unsupported version": good[:4] + (7).to_bytes(4, "little") + good[8:],
        "unknown kind": good[:8] + bytes([5]) + good[9:],
        "truncated payload": good[:-8],
        "trailing bytes": good + b"\0",
        "tag-length mismatch": batch[:-1],
        "invalid modality tag": batch[:-1] + bytes([2]),
        "non-finite": good[:25] + np.array([np.nan]).tobytes() + good[33:],
    }
    for msg, raw in cases.items():
        with pytest.raises(pkg.TensorFormatError, match=msg):
            pkg.load_tensor(_corrupt(tmp_path, raw))
        assert issubclass(pkg.TensorFormatError, ValueError)


def test_layer_directory_round_trip(tmp_path):
    layer = pkg.load_layer(MAN)
    assert layer.use_cws and layer.use_mac and layer.d_out == 40
    out = tmp_path / "again"
    pkg.save_layer(layer, str(out))
    man = json.load(open(MAN))
    files = ["manifest.json"] + [f for f in os.listdir(GOLD) if f.endswith(".spqt") and f not in
                                 ("batch.spqt", "matrix.spqt")]
    for f in files:
        assert filecmp.cmp(out / f, os.path.join(GOLD, f), shallow=False), f
    assert man["format"] == "modquant-layer"
    with pytest.raises(ValueError, match="not a layer manifest"):
        bad = tmp_path / "m.json"
        bad.write_text(json.dumps({"format": "x"}))
        pkg.load_layer(str(bad))


def test_packed_blob_round_trip(tmp_path):
    layer = pkg.load_layer(MAN)
    ref = runtime.pack_arrays(layer)
    path = pkg.save_packed(layer, str(tmp_path / "p.npz"), source_hash="abc")
    got = layer_io.read_packed(path)
    assert str(got["source_hash"]) == "abc"
    for k, v in ref.items():
        np.testing.assert_array_equal(got[k], v, err_msg=k)
        assert got[k].dtype == v.dtype, k
    assert ref["q_main"].dtype == np.int8 and int(ref["use_cws"]) == 1 and int(ref["r_mac"]) > 0
    np.savez(tmp_path / "foreign.npz", format=np.array("other"), version=np.array(1))
    with pytest.raises(ValueError, match="not a splitq packed layer"):
        layer_io.read_packed(str(tmp_path / "foreign.npz"))


def test_dir_hash_tracks_content(tmp_path):
    d = tmp_path / "L"
    shutil.copytree(GOLD, d)
    h0 = layer_io._dir_hash(str(d / "manifest.json"))
    (d / "matrix.spqt").write_bytes(b"unrelated")  # not named by the manifest
    assert layer_io._dir_hash(str(d / "manifest.json")) == h0
    w = pkg.load_tensor(str(d / "w_main.spqt"))
    w[0, 0] += 1.0
    pkg.save_tensor(str(d / "w_main.spqt"), w)
    assert layer_io._dir_hash(str(d / "manifest.json")) != h0
