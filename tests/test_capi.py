"""The C-ABI shared library builds, loads and exports every entry point
include/splitq.h declares (no compute without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    text = open(os.path.join(ROOT, "include", "splitq.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(splitq_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    fns = _header_functions()
    for need in ("splitq_layer_create", "splitq_forward", "splitq_quantize_rows",
                 "splitq_mocd_absmax", "splitq_mocd_rank_counts", "splitq_mocd_text_score"):
        assert need in fns


def test_library_exports_every_declared_symbol():
    from paper_2605_19929_b200 import _lib
    lib = _lib.load()
    for name in _header_functions():
        assert hasattr(lib, name), f"{name} declared in splitq.h but not exported"
    assert set(_lib.EXPORTED_SYMBOLS) <= set(_header_functions())
    assert lib.splitq_version() >= 1


def test_library_is_sm100a_code():
    from paper_2605_19929_b200 import _lib
    path = _lib.lib_path()
    data = open(path, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_invalid_arguments_map_to_valueerror():
    from paper_2605_19929_b200 import _lib
    lib = _lib.load()
    with pytest.raises(ValueError):
        _lib.check(lib.splitq_layer_create(None, 0, ctypes.byref(ctypes.c_void_p())))
    lay = _lib.WsLayout()
    with pytest.raises(ValueError, match="at least one token"):
        _lib.check(lib.splitq_workspace_layout(ctypes.c_void_p(1), 0, ctypes.byref(lay)))


def test_unsupported_spec_rejected_before_any_device_work():
    """bits outside 2..8 and identity specs are refused with ValueError
    (quantizer.py:33-39; the 16-bit / identity cases stay on the CPU)."""
    import numpy as np
    from paper_2605_19929_b200 import _lib
    lib = _lib.load()
    d = _lib.LayerDesc()
    d.d_in, d.d_out, d.n_main = 4, 4, 4
    cm = np.arange(4, dtype=np.int64)
    d.c_main = cm.ctypes.data_as(ctypes.c_void_p)
    d.act = _lib.QSpec(16, 0)
    d.weight = _lib.QSpec(4, 1)
    with pytest.raises(ValueError, match="2..8"):
        _lib.check(lib.splitq_layer_create(ctypes.byref(d), 0, ctypes.byref(ctypes.c_void_p())))
