import sys, torch, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2201_02791_b200 import _lib
lib = _lib.require_cuda()
torch.manual_seed(0)
M, K, N = 1000, 100, 200
A = torch.randn(M, K, device="cuda"); B = torch.randn(K, N, device="cuda")
def gemm(A, B):
    C = torch.zeros(A.shape[0], B.shape[1], device="cuda")
    ws = torch.empty(lib.kg_gemm_workspace_bytes(A.shape[0], K, B.shape[1]), dtype=torch.uint8, device="cuda")
    _lib.call("kg_gemm_f32", A.data_ptr(), K, None, B.data_ptr(), B.shape[1], C.data_ptr(), B.shape[1], None,
              A.shape[0], K, B.shape[1], 0, 0, 0, ws.data_ptr(), ws.numel(), _lib.stream_handle())
    return C
C = gemm(A, B)
pr = torch.randperm(M, device="cuda"); pc = torch.randperm(N, device="cuda")
C2 = gemm(A[pr].contiguous(), B[:, pc].contiguous())
back = torch.empty_like(C2); back[pr] = C2
back2 = torch.empty_like(back); back2[:, pc] = back
print("bitwise equal after un-permuting:", torch.equal(back2, C), "max diff", (back2 - C).abs().max().item())
# single row/col extraction
C3 = gemm(A[5:6].contiguous(), B[:, 7:8].repeat(1, 16).contiguous())
print("single element equal:", C3[0, 0].item() == C[5, 7].item(), C3[0,0].item(), C[5,7].item())
