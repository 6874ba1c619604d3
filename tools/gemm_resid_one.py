"""Run the fused-residual GEMM (C = A B + bias + R) a few times (for ncu).
usage: python tools/gemm_resid_one.py M N K"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1804_00344_b200 import cabi

M, N, K = (int(x) for x in sys.argv[1:4])
A = torch.randn(M, K, device="cuda")
B = torch.randn(K, N, device="cuda")
C = torch.empty(M, N, device="cuda")
R = torch.randn(M, N, device="cuda")
bias = torch.randn(N, device="cuda")
ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    cabi.gemm(M, N, K, A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, precision=1, beta=1.0,
              bias=bias.data_ptr(), addend=R.data_ptr(), workspace=ws.data_ptr(),
              workspace_bytes=ws.numel(), stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
