"""The custom ops' fake (meta) implementations: shapes and dtypes propagate
under FakeTensorMode without a GPU (what torch.compile traces)."""

import pytest

torch = pytest.importorskip("torch")


def test_quantize_op_fake_shapes():
    from torch._subclasses.fake_tensor import FakeTensorMode
    from paper_2605_19929_b200 import ops  # noqa: F401  (registers torch.ops.splitq.*)
    with FakeTensorMode():
        x = torch.empty(5, 37, dtype=torch.float16, device="cuda")
        codes, s, z, st = torch.ops.splitq.quantize_per_token(x, 4, False)
    assert codes.shape == (5, 48) and codes.dtype == torch.int8
    assert s.shape == (5,) and s.dtype == torch.float64
    assert z.dtype == torch.int32 and st.shape == (4,)


def test_ops_registered():
    from paper_2605_19929_b200 import ops  # noqa: F401
    assert hasattr(torch.ops.splitq, "forward")
    assert hasattr(torch.ops.splitq, "quantize_per_token")


def test_top_level_exports_match_reference_mocd_api():
    """modquant/__init__.py:20-30 exports the MOCD functions at top level."""
    import paper_2605_19929_b200 as pkg
    for name in ("build_partition", "vision_score", "percentile_rank", "text_score", "select_topk",
                 "jaccard", "MocdConfig", "ChannelPartition", "stability_report"):
        assert hasattr(pkg, name), name
