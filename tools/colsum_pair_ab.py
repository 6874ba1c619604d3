"""A/B of the fused-operand-sum dW products with / without CTA pairs.
usage: python tools/colsum_pair_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1804_00344_b200 import cabi

ws = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for M, N, K, which in [(2048, 512, 6500, "B"), (512, 2048, 6500, "B"), (32000, 512, 6500, "A"),
                       (2048, 512, 6500, None), (32000, 512, 6500, None)]:
    dy_cols = N if which != "A" else M
    x_cols = M if which != "A" else N
    Dy = torch.randn(K, dy_cols, device="cuda")
    X = torch.randn(K, x_cols, device="cuda")
    A, B = (X, Dy) if which != "A" else (Dy, X)
    lda, ldb = (x_cols, dy_cols) if which != "A" else (dy_cols, x_cols)
    cs = torch.zeros(dy_cols, device="cuda")
    Cd = torch.zeros(M, N, device="cuda")
    res = {}
    for rnd in range(2):
        for mode in (1, 3, 0):
            cabi.lib().mtkc_gemm_set_pair(mode)

            def run():
                kw = {} if which is None else dict(colsum=cs.data_ptr(), colsum_of=2 if which == "B" else 1)
                cabi.gemm(M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, Cd.data_ptr(), N, trans_a=True,
                          precision=1, workspace=ws.data_ptr(), workspace_bytes=ws.numel(), stream=st, **kw)
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                run()
            e1.record()
            torch.cuda.synchronize()
            res[mode] = min(res.get(mode, 1e9), e0.elapsed_time(e1) / 20 * 1e3)
    print(f"M{M} N{N} K{K} colsum {which}:  pair+cs {res[1]:7.1f}  pair {res[3]:7.1f}  single {res[0]:7.1f} us",
          flush=True)
