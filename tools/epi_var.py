"""Epilogue-variant A/B on one GEMM shape (pair vs single CTA tiles).
usage: python tools/epi_var.py M N K [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1804_00344_b200 import cabi

M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 30
A = torch.randn(M, K, device="cuda")
B = torch.randn(K, N, device="cuda")
C = torch.zeros(M, N, device="cuda")
bias = torch.randn(N, device="cuda")
res = torch.randn(M, N, device="cuda")
mask = torch.zeros(M * ((N + 31) // 32), dtype=torch.int32, device="cuda")
ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
variants = {
    "plain": {},
    "bias": {"bias": bias.data_ptr()},
    "relu": {"relu": True},
    "bias+relu": {"bias": bias.data_ptr(), "relu": True},
    "bias+relu+mask": {"bias": bias.data_ptr(), "relu": True, "relu_mask_out": mask.data_ptr()},
    "bias+resid": {"bias": bias.data_ptr(), "beta": 1.0, "addend": res.data_ptr()},
}
for name, kw in variants.items():
    best = {}
    for rnd in range(2):
        for mode in (1, 0):
            cabi.lib().mtkc_gemm_set_pair(mode)

            def run():
                cabi.gemm(M, N, K, A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, precision=1,
                          workspace=ws.data_ptr(), workspace_bytes=ws.numel(), stream=st, **kw)
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            best[mode] = min(best.get(mode, 1e9), e0.elapsed_time(e1) / reps * 1e3)
    print(f"{name:16s} pair {best[1]:7.1f} us  single {best[0]:7.1f} us", flush=True)
