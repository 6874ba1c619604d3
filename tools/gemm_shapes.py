"""Time arbitrary GEMM shapes: python tools/gemm_shapes.py M,N,K,ta,tb[,beta] ..."""
import os, sys
sys.path.insert(0, os.environ.get("MTK_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1804_00344_b200 import cabi
ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for spec in sys.argv[1:]:
    f = spec.split(",")
    M, N, K, ta, tb = (int(x) for x in f[:5])
    beta = float(f[5]) if len(f) > 5 else 0.0
    A = torch.randn((K, M) if ta else (M, K), device="cuda")
    B = torch.randn((N, K) if tb else (K, N), device="cuda")
    C = torch.zeros(M, N, device="cuda")
    run = lambda: cabi.gemm(M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], C.data_ptr(), N,
                            trans_a=ta, trans_b=tb, beta=beta, precision=1, workspace=ws.data_ptr(),
                            workspace_bytes=ws.numel(), stream=st)
    for _ in range(3): run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    print(f"{spec:28s} {ms*1e3:8.1f} us  {2*M*N*K/ms/1e9:7.1f} TF/s")
