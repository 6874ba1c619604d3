"""Micro-benchmark of mtkc_gemm on the Transformer-base step's GEMM shapes.
usage: python tools/gemm_bench.py [reps]"""
import os
import sys

sys.path.insert(0, os.environ.get("MTK_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1804_00344_b200 import cabi
print("# lib", cabi.LIB_PATH)

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
R = int(os.environ.get("MTK_BENCH_ROWS", "8184"))
shapes = [  # (name, M, N, K, transA, transB)
    ("logits fwd  H.E^T", R, 32000, 512, 0, 1),
    ("logits dH = dL.E", R, 512, 32000, 0, 0),
    ("logits dE = dL^T.H", 32000, 512, R, 1, 0),
    ("proj fwd x.W", R, 512, 512, 0, 0),
    ("proj dX = dY.W^T", R, 512, 512, 0, 1),
    ("proj dW = X^T.dY", 512, 512, R, 1, 0),
    ("ffn1 fwd", R, 2048, 512, 0, 0),
    ("ffn2 dX", R, 2048, 512, 0, 1),
    ("ffn1 dW", 512, 2048, R, 1, 0),
    ("square 8192", 8192, 8192, 8192, 0, 0),
    ("logits fwd +bias", R, 32000, 512, 0, 1, "bias"),
    ("ffn1 fwd +bias+relu", R, 2048, 512, 0, 0, "relu"),
    ("ffn2 dX +gate", R, 2048, 512, 0, 1, "gate"),
    ("proj dW beta=1", 512, 512, R, 1, 0, "beta"),
    ("proj fwd +b+resid", R, 512, 512, 0, 0, "addend"),
    ("ffn2 fwd +b+resid", R, 512, 2048, 0, 0, "addend"),
    ("ffn1 dW +colsum", 512, 2048, R, 1, 0, "colsum"),
]
if os.environ.get("MTK_BENCH_ONLY"):
    keep = os.environ["MTK_BENCH_ONLY"].split(",")
    shapes = [s for s in shapes if any(k in s[0] for k in keep)]
ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream().cuda_stream
for name, M, N, K, ta, tb, *extra in shapes:
    A = torch.randn((K, M) if ta else (M, K), device="cuda")
    B = torch.randn((N, K) if tb else (K, N), device="cuda")
    C = torch.zeros(M, N, device="cuda")
    args = dict(trans_a=ta, trans_b=tb, precision=1, workspace=ws.data_ptr(),
                workspace_bytes=ws.numel(), stream=stream)
    ep = extra[0] if extra else None
    bias = torch.randn(N, device="cuda")
    gate = torch.randn(M, N, device="cuda")
    if ep in ("bias", "relu"):
        args["bias"] = bias.data_ptr()
    if ep == "relu":
        args["relu"] = True
    if ep == "gate":
        args["gate"] = gate.data_ptr()
    if ep == "beta":
        args["beta"] = 1.0
    if ep == "addend":
        addend = torch.randn(M, N, device="cuda")
        args["bias"] = bias.data_ptr()
        args["beta"] = 1.0
        args["addend"] = addend.data_ptr()
    if ep == "colsum":
        cs = torch.zeros(N, device="cuda")
        args["colsum"] = cs.data_ptr()
        args["colsum_of"] = 2  # MTKC_COLSUM_B
    def run():
        cabi.gemm(M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], C.data_ptr(), N, **args)

    modes = [1, 0] if os.environ.get("MTK_BENCH_AB") else [None]
    best = {}
    for rnd in range(2 if modes[0] is not None else 1):
        for mode in modes:
            if mode is not None:
                cabi.lib().mtkc_gemm_set_pair(mode)
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            best[mode] = min(best.get(mode, 1e9), ms)
    ref = (A.t() if ta else A) @ (B.t() if tb else B)
    err = ((C - ref).abs().max() / ref.abs().max()).item() if not ep else float("nan")
    line = f"{name:22s} M{M:6d} N{N:6d} K{K:6d}"
    for mode, ms in best.items():
        tf = 2.0 * M * N * K / ms / 1e9
        tag = "" if mode is None else ("pair " if mode else "single ")
        line += f"  {tag}{ms*1e3:8.1f} us {tf:6.1f} TF/s"
    print(line + f"  relerr {err:.1e}", flush=True)
