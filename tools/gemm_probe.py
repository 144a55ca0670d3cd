"""Standalone timing of the NN GEMM at the FB15k-shape layer sizes through
kg_gemm_f32 (pack + tcgen05 GEMM); run under ncu for per-kernel durations,
KG_GEMM_EXP=1/2/3 drops the epilogue stores / the MMAs / both (diagnostics; tools/r3_gemm_probe.sh)."""
import sys
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2201_02791_b200 import _lib  # noqa: E402

lib = _lib.require_cuda()
for (M, K, N) in [(14541, 200, 100), (14541, 100, 200), (9728, 200, 100)]:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(K, N, device="cuda")
    C = torch.zeros(M, N, device="cuda")
    ws = torch.empty(lib.kg_gemm_workspace_bytes(M, K, N), dtype=torch.uint8, device="cuda")
    rows = torch.randperm(M, device="cuda").to(torch.int32)
    for _ in range(3):
        _lib.call("kg_gemm_f32", A.data_ptr(), K, None, B.data_ptr(), N, C.data_ptr(), N, rows.data_ptr(), M, K, N,
                  1, 0, 0, ws.data_ptr(), ws.numel(), _lib.stream_handle())
    torch.cuda.synchronize()
print("ok")
