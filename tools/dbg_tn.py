import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2201_02791_b200 import _lib
lib = _lib.require_cuda()
for (M, K, N) in [(16, 16, 16), (32, 16, 16), (1000, 128, 256)]:
    A = torch.randn(M, K, device="cuda"); B = torch.randn(M, N, device="cuda")
    ws = torch.empty(lib.kg_gemm_workspace_bytes(M, K, N), dtype=torch.uint8, device="cuda")
    for impl in (0, 2):
        C = torch.zeros((K, N), device="cuda")
        _lib.call("kg_gemm_f32", A.data_ptr(), K, None, B.data_ptr(), N, C.data_ptr(), N, None, M, K, N, 0, 1, impl,
                  ws.data_ptr(), ws.numel(), _lib.stream_handle())
        torch.cuda.synchronize()
        want = A.double().T @ B.double()
        print(M, K, N, impl, float((C.double() - want).abs().max()), float(C.abs().max()), float(want.abs().max()))
