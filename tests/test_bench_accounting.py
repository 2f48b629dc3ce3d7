"""The bench's roofline accounting (CPU): the algorithmic work figures that
bench.py divides by measured times must be SURVEY §8(d)'s."""

import bench
import workloads as wl


def test_prefill_ops_per_token_7b():
    # 2 * D_in * D_out summed over q, k, v, o, gate, up, down: 466,092,032 ops/token
    ops = sum(2 * sp.d_in * sp.d_out for sp in wl.model_specs(wl.QWEN_7B, abits=4))
    assert ops == 466_092_032


def test_decode_weight_bytes_7b():
    # W4 ~124.8 MB, W3 ~96.1 MB per 7B layer
    for wbits, mb in ((4, 124.8), (3, 96.1)):
        alg = sum(bench.decode_weight_bytes(sp, 448, wbits)[0]
                  for sp in wl.model_specs(wl.QWEN_7B, abits=4, wbits=wbits))
        assert abs(alg / 1e6 - mb) < 0.1
    # what the kernels stream (4-bit containers + fp16 aux operand) is never less
    for sp in wl.model_specs(wl.QWEN_7B, abits=4):
        alg, streamed = bench.decode_weight_bytes(sp, 448, 4)
        assert streamed >= alg * 0.99


def test_decode_cli_flags():
    import sys
    argv = sys.argv
    try:
        sys.argv = ["bench.py", "--decode", "--batch", "16", "--wbits", "3", "--abits", "3"]
        a = bench.parse()
    finally:
        sys.argv = argv
    assert a.decode and a.batch == 16 and a.wbits == 3 and a.abits == 3
