"""A/B of the loading epilogues (fused residual, accumulate, ReLU gate) on
the base step's shapes.  usage: [MTK_PKG_ROOT=...] python tools/epi_ab.py"""
import os
import sys

sys.path.insert(0, os.environ.get("MTK_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1804_00344_b200 import cabi

R = 8184
ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cases = [("oproj fwd +bias", R, 512, 512, 0, {}), ("oproj fwd +bias+resid", R, 512, 512, 0, {"res": 1}),
         ("ffn2 fwd +bias", R, 512, 2048, 0, {}), ("ffn2 fwd +bias+resid", R, 512, 2048, 0, {"res": 1}),
         ("ffn2 dX", R, 2048, 512, 1, {"nobias": 1}), ("ffn2 dX +gate", R, 2048, 512, 1, {"gate": 1, "nobias": 1}),
         ("proj dX beta=1", R, 512, 512, 1, {"beta": 1, "nobias": 1})]
for name, M, N, K, tb, kw in cases:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda") if tb else torch.randn(K, N, device="cuda")
    C = torch.zeros(M, N, device="cuda")
    bias = torch.randn(N, device="cuda")
    res = torch.randn(M, N, device="cuda")
    gate = torch.randn(M, N, device="cuda")

    def run():
        cabi.gemm(M, N, K, A.data_ptr(), K, B.data_ptr(), K if tb else N, C.data_ptr(), N,
                  trans_b=bool(tb), beta=1.0 if (kw.get("res") or kw.get("beta")) else 0.0,
                  bias=None if kw.get("nobias") else bias.data_ptr(),
                  addend=res.data_ptr() if kw.get("res") else None,
                  gate=gate.data_ptr() if kw.get("gate") else None,
                  workspace=ws.data_ptr(), workspace_bytes=ws.numel())
    for _ in range(3):
        run()
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{name:24s} M{M} N{N} K{K}: {ts[len(ts) // 2]:.1f} us", flush=True)
