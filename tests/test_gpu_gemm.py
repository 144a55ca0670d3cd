"""tcgen05 3xTF32 GEMMs (the factored-layer contractions) vs a float64
reference through the C ABI — B200 only. Tolerance: max |err| / max |ref|
<= 5e-6 (3xTF32 ~ fp32 accuracy; plain TF32 would be ~1e-3)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2201_02791_b200 import _lib  # noqa: E402


def run(A, B, M, K, N, a_rows=None, c_rows=None, relu=0, trans=0, impl=0, C=None):
    lib = _lib.require_cuda()
    ws = torch.empty(lib.kg_gemm_workspace_bytes(max(M, 1), K, N), dtype=torch.uint8, device="cuda")
    if C is None:
        C = torch.zeros((K, N) if trans else (M if c_rows is None else int(c_rows.max()) + 1, N),
                        dtype=torch.float32, device="cuda")
    _lib.call("kg_gemm_f32", A.data_ptr(), A.shape[1], _lib.ptr(a_rows), B.data_ptr(), B.shape[1], C.data_ptr(),
              C.shape[1], _lib.ptr(c_rows), M, K, N, relu, trans, impl, ws.data_ptr(), ws.numel(),
              _lib.stream_handle())
    torch.cuda.synchronize()
    return C


def err(got, want):
    return float((got.double() - want).abs().max() / max(want.abs().max().item(), 1e-30))


@pytest.mark.parametrize("M,K,N", [(1000, 200, 100), (14541, 100, 200), (300, 5, 6), (5, 3, 4), (130, 256, 256),
                                   (257, 33, 17), (1, 8, 16),
                                   # fp32 A records (> 65,536 rows): weight-resident CTA pairs for N % 32 == 0
                                   (70001, 128, 256), (70001, 256, 128), (70001, 100, 64), (70001, 100, 100)])
@pytest.mark.parametrize("impl", [0, 1])
def test_nn_gathered_rows(M, K, N, impl):
    g = torch.Generator(device="cuda").manual_seed(M + K + N)
    src_rows = M + 37
    A = torch.randn(src_rows, K, device="cuda", generator=g)
    B = torch.randn(K, N, device="cuda", generator=g)
    a_rows = torch.randperm(src_rows, device="cuda", generator=g)[:M].to(torch.int32)
    c_rows = torch.randperm(M + 11, device="cuda", generator=g)[:M].to(torch.int32)
    C = run(A, B, M, K, N, a_rows, c_rows, relu=1, impl=impl)
    want = torch.relu(A.double()[a_rows.long()] @ B.double())
    assert err(C[c_rows.long()], want) < 5e-6


@pytest.mark.parametrize("M,K,N", [(14541, 100, 200), (1000, 128, 256), (50, 3, 8), (3000, 200, 64), (7, 5, 6),
                                   (70001, 128, 256), (70001, 32, 64)])
@pytest.mark.parametrize("impl", [0, 1, 2])
def test_tn_reduction(M, K, N, impl):
    """impl 2: the record TN (X / dS operand records read as MN-major
    operands, split hi|lo records below 65,536 rows, fp32 records above)."""
    if impl == 2 and K > 128:
        pytest.skip("record TN: d_in <= 128")
    g = torch.Generator(device="cuda").manual_seed(7 * M + K)
    A = torch.randn(M + 5, K, device="cuda", generator=g)
    Bm = torch.randn(M, N, device="cuda", generator=g)
    a_rows = torch.randperm(M + 5, device="cuda", generator=g)[:M].to(torch.int32)
    C = run(A, Bm, M, K, N, a_rows, trans=1, impl=impl)
    want = A.double()[a_rows.long()].T @ Bm.double()
    assert err(C, want) < 5e-6
