"""The A2 x W3 / W2 prefill main GEMM on tcgen05 kind::mxf4 (E2M1 codes, unit
UE8M0 block scales): A2 codes (q - zp in [-3, 3]) and
W3 / W2 codes are exact in E2M1 and their products are small integers, so
the fp32 accumulator must hold exactly the int32 sum the int8 path
produces. Checked against the oracle (codes and the int32 main accumulator
bit-exact, outputs within 1e-3 rms) and against the int8 path
(SPLITQ_NO_MXF4=1): main accumulators and outputs bit-identical."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from test_gpu_forward import _case, _check_acc, _check_codes, _check_out  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = {  # > 2048 rows: the prefill tcgen05 path
    "a2w3": dict(seed=31, T=2600, d_in=512, d_out=384, k_t=8, k_v=8, r_s=4, r_c=6, abits=2, wbits=3),
    "a2w3_f16": dict(seed=32, T=3000, d_in=1024, d_out=200, k_t=16, k_v=16, r_s=8, r_c=8, abits=2, wbits=3,
                     x_dtype=np.float16),
    "a2w2": dict(seed=33, T=2100, d_in=384, d_out=160, k_t=8, k_v=8, r_s=4, r_c=4, abits=2, wbits=2),
    "a2w3_no_aux": dict(seed=34, T=2500, d_in=512, d_out=512, k_t=0, k_v=0, r_s=0, r_c=0, abits=2, wbits=3),
    "a2w3_sym": dict(seed=35, T=2300, d_in=640, d_out=256, k_t=8, k_v=8, r_s=4, r_c=4, abits=2, wbits=3,
                     a_sym=True),
    "a2w3_wide_k": dict(seed=36, T=2200, d_in=4096, d_out=128, k_t=32, k_v=32, r_s=8, r_c=8, abits=2, wbits=3),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_mxf4_against_oracle(name):
    layer, x, tags = _case(**CASES[name])
    _check_codes(layer, x, tags)
    _check_acc(layer, x, tags)
    _check_out(layer, x, tags)


@pytest.mark.parametrize("name", sorted(CASES))
def test_mxf4_equals_int8_path(name, monkeypatch):
    from paper_2605_19929_b200 import runtime
    layer, x, tags = _case(**CASES[name])
    g = runtime.packed(layer)
    assert g.layout(x.shape[0]).a_main_fp4 >= 0, "layer should take the kind::mxf4 path"
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(tags).cuda()
    raw_a, y_a = g.run(xd, td, raw=True).cpu().numpy(), g.run(xd, td).cpu().numpy()
    monkeypatch.setenv("SPLITQ_NO_MXF4", "1")
    raw_b, y_b = g.run(xd, td, raw=True).cpu().numpy(), g.run(xd, td).cpu().numpy()
    np.testing.assert_array_equal(raw_a[0], raw_b[0])
    # outputs: same main accumulator; the fp32 aux plane may be summed in
    # another order when the two paths split K differently (small calls)
    np.testing.assert_allclose(y_a, y_b, rtol=1e-5, atol=1e-5 * np.abs(y_b).max())


def test_a3_layers_stay_on_int8():
    """A3 codes (q - zp up to 7) are not all E2M1 values: no fp4 copy."""
    from paper_2605_19929_b200 import runtime
    layer, x, tags = _case(seed=37, T=2100, d_in=512, d_out=128, k_t=8, k_v=8, r_s=4, r_c=4, abits=3, wbits=3)
    assert runtime.packed(layer).layout(x.shape[0]).a_main_fp4 < 0
