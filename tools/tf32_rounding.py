"""Does the tcgen05 kind::tf32 path truncate fp32 operands (RZ) or round them?
Compares the device product of raw fp32 operands with host products of
operands pre-rounded to tf32 by truncation and by round-to-nearest."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1804_00344_b200 import cabi

def trunc(x):
    u = x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return u.view(np.float32)

def rna(x):
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x1000) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)

def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()

rng = np.random.default_rng(0)
M, K, N = 512, 1024, 512
a = rng.standard_normal((M, K)).astype(np.float32)
b = rng.standard_normal((K, N)).astype(np.float32)
exact = a.astype(np.float64) @ b.astype(np.float64)
for name, (x, y) in {"raw": (a, b), "pre_trunc": (trunc(a), trunc(b)), "pre_rna": (rna(a), rna(b))}.items():
    A, B = dev(x), dev(y)
    C = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    path = cabi.gemm(M, N, K, A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, precision=1)
    torch.cuda.synchronize()
    c = C.cpu().numpy().astype(np.float64)
    e = c - exact
    slope = float(np.sum(e * exact) / np.sum(exact * exact))
    rms = float(np.sqrt(np.mean(e * e)) / np.sqrt(np.mean(exact * exact)))
    hx = x.astype(np.float64) @ y.astype(np.float64)
    print(f"{name:10s} path {path} slope {slope:+.3e} rel-rms {rms:.3e}  "
          f"max|dev - host(pre-rounded operands)| {np.abs(c - hx).max():.3e}")
