"""A/B of the fused bias-gradient sums on the dW GEMM shapes of the base step:
plain dW, dW + fused colsum, dW + separate mtkc_colsum (MTK_NO_FUSED_COLSUM).
usage: [MTK_CS_DIST=0] python tools/colsum_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1804_00344_b200 import cabi

R = 8184
shapes = [("proj dW", 512, 512, R, 2), ("ffn1 dW", 512, 2048, R, 2), ("ffn2 dW", 2048, 512, R, 2),
          ("logits dE", 32000, 512, R, 1)]
ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, M, N, K, which in shapes:
    A = torch.randn(K, M, device="cuda")
    B = torch.randn(K, N, device="cuda")
    C = torch.zeros(M, N, device="cuda")
    cs = torch.zeros(N if which == 2 else M, device="cuda")
    res = []
    for mode in ("plain", "fused"):
        def run():
            cabi.gemm(M, N, K, A.data_ptr(), M, B.data_ptr(), N, C.data_ptr(), N, trans_a=True,
                      workspace=ws.data_ptr(), workspace_bytes=ws.numel(),
                      colsum=cs.data_ptr() if mode == "fused" else None, colsum_of=which)
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
        res.append(f"{mode} {ts[len(ts) // 2]:.1f}us")
    print(f"{name:10s} M{M} N{N} K{K}: " + "  ".join(res), flush=True)
