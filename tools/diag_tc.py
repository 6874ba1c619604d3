import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1804_00344_b200 import cabi

def run(M, N, K, ta, tb, seed=0):
    rng = np.random.default_rng(seed)
    a = rng.integers(-2, 3, (K, M) if ta else (M, K)).astype(np.float32)
    b = rng.integers(-2, 3, (N, K) if tb else (K, N)).astype(np.float32)
    A = torch.from_numpy(a).cuda(); B = torch.from_numpy(b).cuda()
    C = torch.zeros(M, N, device="cuda")
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    path = cabi.gemm(M, N, K, A.data_ptr(), a.shape[1], B.data_ptr(), b.shape[1], C.data_ptr(), N,
                     trans_a=ta, trans_b=tb, precision=1, workspace=ws.data_ptr(), workspace_bytes=ws.numel())
    torch.cuda.synchronize()
    got = C.cpu().numpy()
    opa = a.T if ta else a; opb = b.T if tb else b
    ex = opa @ opb
    err = np.abs(got - ex).max()
    # probe alternative interpretations
    alts = {}
    alts["zero"] = np.abs(got).max()
    return path, err, alts

for env in ["1", "0"]:
    os.environ["MTK_TMA_TF32"] = env
    for (M, N, K) in [(128, 128, 8), (128, 128, 32), (128, 128, 64), (256, 256, 96)]:
        for ta in (0, 1):
            for tb in (0, 1):
                p, e, alts = run(M, N, K, ta, tb)
                print(f"tf32round={env} M{M} N{N} K{K} ta{ta} tb{tb} path{p} maxerr {e:.3g} maxabs {alts['zero']:.3g}", flush=True)
    break
