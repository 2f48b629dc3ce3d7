"""Layer state on disk: the reference's calibrated-layer
directory (manifest.json + SPQT tensors), read straight into a packed device
layer, plus a packed blob that skips the weight quantization on reload.

Mirrors (same names, layout and errors):
  * ``save_tensor`` / ``load_tensor``  -- reference tensor.py:118-170, the
    SPQT dump: magic "SPQT", u32 version, u8 kind (0 matrix, 1 batch), u64
    rows, u64 cols, rows*cols little-endian float64 row-major, then one tag
    byte per row for batches. Errors: ``TensorFormatError`` (a ValueError).
  * ``save_layer`` / ``load_layer``    -- reference layer.py:237-352, the
    directory of SPQT files plus a JSON manifest ("modquant-layer", v1).

Beyond the reference (it re-quantizes the weights on every forward, F5, and
has no packed format):
  * ``save_packed(layer, path)`` writes what ``splitq_layer_create`` consumes
    -- partition, smoothing scales, the integer weight codes and fp64 column
    scales of Q(R), Q(W_t/d_t), Q(W_v/d_v), Q(u*), Q(gate v) and the spec
    words -- as an uncompressed ``.npz`` ("splitq-packed", v1). The codes
    are computed on the host with the reference's own numpy expressions
    (runtime.pack_arrays), so a reload is bit-identical to packing afresh.
  * ``load_packed(path)`` -> ``runtime.GpuLayer`` without recomputing codes.
  * ``load_layer_packed(manifest)`` -> ``GpuLayer``; caches the packed blob
    next to the manifest, keyed by a hash of the manifest and its tensors.
"""

from __future__ import annotations

import hashlib
import json
import os
import struct

import numpy as np

from . import lowrank
from . import transform as tr
from .layer import SplitLayer
from .mocd import ChannelPartition
from .quantizer import Granularity, QuantSpec
from .tensor import ActivationBatch, as_matrix

MAGIC = b"SPQT"
FORMAT_VERSION = 1
_KIND_MATRIX = 0
_KIND_BATCH = 1
_HEADER = "<IBQQ"
PACKED_FORMAT = "splitq-packed"
PACKED_VERSION = 1
PACKED_NAME = "splitq_packed.npz"


class TensorFormatError(ValueError):  # tensor.py:23-24
    """A malformed SPQT dump."""


# ---------------------------------------------------------------- SPQT tensors
def save_tensor(path, obj) -> None:
    """Write a matrix or ActivationBatch as an SPQT dump (tensor.py:118-135)."""
    if isinstance(obj, ActivationBatch):
        data = np.asarray(obj.data, dtype=np.float64)
        tags = np.asarray(obj.tags, dtype=np.uint8)
        kind = _KIND_BATCH
    else:
        data, tags, kind = as_matrix(obj), None, _KIND_MATRIX
    rows, cols = data.shape
    with open(path, "wb") as fh:
        fh.write(MAGIC + struct.pack(_HEADER, FORMAT_VERSION, kind, rows, cols))
        fh.write(np.ascontiguousarray(data, dtype="<f8").tobytes())
        if tags is not None:
            fh.write(tags.tobytes())


def load_tensor(path):
    """Read an SPQT dump (tensor.py:138-170): a float64 matrix, or an
    ActivationBatch when the dump carries tags."""
    with open(path, "rb") as fh:
        raw = fh.read()
    hsz = struct.calcsize(_HEADER)
    if len(raw) < len(MAGIC) + hsz:
        raise TensorFormatError("truncated header")
    if raw[:4] != MAGIC:
        raise TensorFormatError("bad magic")
    version, kind, rows, cols = struct.unpack_from(_HEADER, raw, 4)
    if version != FORMAT_VERSION:
        raise TensorFormatError(f"unsupported version {version}")
    if kind not in (_KIND_MATRIX, _KIND_BATCH):
        raise TensorFormatError(f"unknown kind {kind}")
    start = 4 + hsz
    nbytes = rows * cols * 8
    if len(raw) < start + nbytes:
        raise TensorFormatError("truncated payload")
    values = np.frombuffer(raw, dtype="<f8", count=rows * cols, offset=start).reshape(rows, cols).copy()
    if not np.all(np.isfinite(values)):
        raise TensorFormatError("non-finite value")
    rest = raw[start + nbytes:]
    if kind == _KIND_MATRIX:
        if rest:
            raise TensorFormatError("trailing bytes after matrix payload")
        return values
    if len(rest) != rows:
        raise TensorFormatError("tag-length mismatch")
    tags = np.frombuffer(rest, dtype=np.uint8).copy()
    if np.any(tags > 1):
        raise TensorFormatError("invalid modality tag")
    return ActivationBatch(values, tags)


# ---------------------------------------------------------------- layer directories
def _spec_dict(spec) -> dict:
    g = spec.granularity
    return {"bits": spec.bits, "symmetric": spec.symmetric, "granularity": getattr(g, "value", g)}


def _spec(d: dict) -> QuantSpec:
    return QuantSpec(d["bits"], d["symmetric"], Granularity(d["granularity"]))


def save_layer(layer, out_dir: str) -> str:
    """Write the layer's tensors and a JSON manifest (layer.py:284-322);
    returns the manifest path. Diagonal transforms only (the GPU path's)."""
    os.makedirs(out_dir, exist_ok=True)
    p = layer.partition
    man = {
        "format": "modquant-layer", "version": 1, "dim": int(p.dim), "d_out": int(layer.w_main.shape[1]),
        "partition": {"c_main": np.asarray(p.c_main).tolist(), "c_text": np.asarray(p.c_text).tolist(),
                      "c_vision": np.asarray(p.c_vision).tolist()},
        "act_spec": _spec_dict(layer.act_spec), "weight_spec": _spec_dict(layer.weight_spec),
        "use_cws": bool(layer.use_cws), "use_mac": bool(layer.use_mac),
        "aux_bits_floor": int(layer.aux_bits_floor),
    }
    for name in ("w_main", "w_text", "w_vision"):
        save_tensor(os.path.join(out_dir, name + ".spqt"), getattr(layer, name))
        man[name] = name + ".spqt"
    for name in ("p_main", "p_text", "p_vision"):
        t = getattr(layer, name)
        if not t.is_diagonal:
            raise ValueError("dense transforms are not supported on the GPU path")
        fname = f"{name}_scale.spqt"
        save_tensor(os.path.join(out_dir, fname), np.asarray(t.scale).reshape(1, -1))
        man[name] = {"kind": "diagonal", "file": fname}
    for name in ("branch_smooth", "branch_comp"):
        br = getattr(layer, name)
        if br is None:
            continue
        files = {}
        for part, value in (("u_star", br.u_star), ("v_base", br.v_base),
                            ("gate", np.asarray(br.gate).reshape(1, -1))):
            fname = f"{name}_{part}.spqt"
            save_tensor(os.path.join(out_dir, fname), value)
            files[part] = fname
        man[name] = files
    path = os.path.join(out_dir, "manifest.json")
    with open(path, "w") as fh:
        json.dump(man, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return path


def _transform(entry: dict, in_dir: str, dim: int) -> tr.Transform:
    data = load_tensor(os.path.join(in_dir, entry["file"]))
    if entry["kind"] != "diagonal":
        raise ValueError("dense transforms are not supported on the GPU path")
    if dim == 0:
        return tr.identity_transform(0)
    return tr.diagonal_transform(np.asarray(data).reshape(-1))


def load_layer(manifest_path: str) -> SplitLayer:
    """Read a layer directory (layer.py:325-352) into a SplitLayer."""
    with open(manifest_path) as fh:
        man = json.load(fh)
    if man.get("format") != "modquant-layer":
        raise ValueError("not a layer manifest")
    d = os.path.dirname(os.path.abspath(manifest_path))
    part = man["partition"]
    partition = ChannelPartition(np.asarray(part["c_main"], np.int64), np.asarray(part["c_text"], np.int64),
                                 np.asarray(part["c_vision"], np.int64), man["dim"])
    kw = {}
    for name in ("branch_smooth", "branch_comp"):
        if name in man:
            e = man[name]
            kw[name] = lowrank.LowRankBranch(load_tensor(os.path.join(d, e["u_star"])),
                                             load_tensor(os.path.join(d, e["v_base"])),
                                             np.asarray(load_tensor(os.path.join(d, e["gate"]))).reshape(-1))
    return SplitLayer(
        partition=partition,
        w_main=load_tensor(os.path.join(d, man["w_main"])),
        w_text=load_tensor(os.path.join(d, man["w_text"])),
        w_vision=load_tensor(os.path.join(d, man["w_vision"])),
        p_main=_transform(man["p_main"], d, len(partition.c_main)),
        p_text=_transform(man["p_text"], d, len(partition.c_text)),
        p_vision=_transform(man["p_vision"], d, len(partition.c_vision)),
        act_spec=_spec(man["act_spec"]), weight_spec=_spec(man["weight_spec"]),
        use_cws=man["use_cws"], use_mac=man["use_mac"], aux_bits_floor=man["aux_bits_floor"], **kw)


# ---------------------------------------------------------------- packed blobs
def save_packed(layer, path: str, source_hash: str = "") -> str:
    """Write the packed layer (runtime.pack_arrays) as an uncompressed .npz."""
    from . import runtime
    arrays = runtime.pack_arrays(layer)
    arrays["format"] = np.array(PACKED_FORMAT)
    arrays["version"] = np.array(PACKED_VERSION)
    arrays["source_hash"] = np.array(source_hash)
    tmp = path + ".tmp.npz"
    np.savez(tmp, **arrays)
    os.replace(tmp, path)
    return path


def read_packed(path: str) -> dict:
    """The arrays of a packed blob (host; no GPU needed)."""
    with np.load(path, allow_pickle=False) as z:
        if str(z["format"]) != PACKED_FORMAT:
            raise ValueError("not a splitq packed layer")
        if int(z["version"]) != PACKED_VERSION:
            raise ValueError(f"unsupported packed version {int(z['version'])}")
        return {k: z[k] for k in z.files}


def load_packed(path: str, dev=None):
    """A GpuLayer from a packed blob, without recomputing the weight codes."""
    from . import runtime
    return runtime.GpuLayer(arrays=read_packed(path), dev=dev)


def _dir_hash(manifest_path: str) -> str:
    """sha256 over the manifest and every file it names (content, not mtime)."""
    d = os.path.dirname(os.path.abspath(manifest_path))
    with open(manifest_path, "rb") as fh:
        raw = fh.read()
    h = hashlib.sha256(raw)
    man = json.loads(raw)

    def files(v):
        if isinstance(v, str) and v.endswith(".spqt"):
            yield v
        elif isinstance(v, dict):
            for x in v.values():
                yield from files(x)

    for f in sorted(set(files(man))):
        with open(os.path.join(d, f), "rb") as fh:
            h.update(f.encode() + b"\0" + hashlib.sha256(fh.read()).digest())
    return h.hexdigest()


def load_layer_packed(manifest_path: str, dev=None, cache: bool = True):
    """A layer directory straight to a packed device layer. With ``cache``,
    the packed blob is kept next to the manifest (splitq_packed.npz) and
    reused while the directory's content hash matches."""
    from . import runtime
    blob = os.path.join(os.path.dirname(os.path.abspath(manifest_path)), PACKED_NAME)
    digest = _dir_hash(manifest_path)
    if cache and os.path.exists(blob):
        try:
            arrays = read_packed(blob)
            if str(arrays["source_hash"]) == digest:
                return runtime.GpuLayer(arrays=arrays, dev=dev)
        except (ValueError, OSError, KeyError):
            pass  # stale or foreign blob: rebuild it
    layer = load_layer(manifest_path)
    if cache:
        save_packed(layer, blob, source_hash=digest)
        return runtime.GpuLayer(arrays=read_packed(blob), dev=dev)
    return runtime.GpuLayer(layer, dev)
