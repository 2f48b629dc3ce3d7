"""tcgen05 kind::i8 GEMM (the forward's main-path kernel in raw mode) is
bit-exact against an int64 host product."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _run(m, n, k, a_signed, seed):
    from paper_2605_19929_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(seed)
    lda = (k + 15) // 16 * 16
    if a_signed:
        a = rng.integers(-128, 128, (m, lda), dtype=np.int64)
    else:
        a = rng.integers(0, 256, (m, lda), dtype=np.int64)
    b = rng.integers(-128, 128, (n, lda), dtype=np.int64)
    a[:, k:] = 0
    b[:, k:] = 0
    a_d = torch.from_numpy(a.astype(np.uint8 if not a_signed else np.int8)).cuda()
    b_d = torch.from_numpy(b.astype(np.int8)).cuda()
    c_d = torch.zeros((m, n), dtype=torch.int32, device="cuda")
    _lib.check(lib.splitq_gemm_i8(a_d.data_ptr(), lda, int(a_signed), b_d.data_ptr(), lda,
                                  c_d.data_ptr(), n, m, n, k, None))
    torch.cuda.synchronize()
    ref = a[:, :k] @ b[:, :k].T
    got = c_d.cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("m,n,k", [(128, 128, 128), (256, 384, 512), (300, 200, 1000),
                                   (77, 16, 32), (1024, 512, 2016), (129, 130, 4096)])
@pytest.mark.parametrize("a_signed", [1, 0])
def test_gemm_i8_exact(m, n, k, a_signed):
    _run(m, n, k, a_signed, seed=m * 7 + n + k)
