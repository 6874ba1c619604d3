"""Run one GEMM shape a few times (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1804_00344_b200 import cabi
M, N, K, ta, tb = (int(x) for x in sys.argv[1:6])
A = torch.randn((K, M) if ta else (M, K), device="cuda")
B = torch.randn((N, K) if tb else (K, N), device="cuda")
C = torch.empty(M, N, device="cuda")
ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    cabi.gemm(M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], C.data_ptr(), N,
              trans_a=ta, trans_b=tb, precision=1, workspace=ws.data_ptr(), workspace_bytes=ws.numel(),
              stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
