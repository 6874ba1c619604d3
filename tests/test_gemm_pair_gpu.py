"""CTA-pair (tcgen05.mma.cta_group::2) tiles of the tensor-core GEMM.

Pairs are chosen for M >= 1024 with more than one wave of single-CTA tiles or
a long k loop.  Every product runs twice -- pairs on (mtkc_gemm_set_pair(1))
and off -- over ragged M / N, all four operand majors and every epilogue the
model uses (bias, ReLU + bit mask, fused residual, beta*C, float gate, gate
bit mask), split-K, problem groups / K-concatenation and the fused operand
sums.  Both must meet the TF32 bound |C - C64| <= 4e-3 (|A||B|)_ij (+ the
epilogue terms), and pairs must not change the result beyond it: the MMA
sums each output's k-range in the same order in both modes, so the two
results are expected to agree bit for bit; the test asserts the bound and
records exact agreement.
"""
import ctypes as C

import numpy as np
import pytest

from paper_1804_00344_b200 import cabi

pytestmark = pytest.mark.gpu


@pytest.fixture
def pair_modes(cuda):
    yield
    cabi.lib().mtkc_gemm_set_pair(1)


def _both(fn, on=1):
    out = {}
    for mode in (on, 0):
        cabi.lib().mtkc_gemm_set_pair(mode)
        out[mode] = fn()
    cabi.lib().mtkc_gemm_set_pair(1)
    return out[on], out[0]


def _tol(a64, b64, extra=0.0):
    return 4e-3 * (np.abs(a64) @ np.abs(b64) + extra)


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("shape", [(1100, 2048, 512), (2048, 520, 2048), (1300, 300, 1024)])
def test_pair_majors(pair_modes, ta, tb, shape):
    import torch
    rng = np.random.default_rng(1)
    M, N, K = shape
    a = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def run():
        Cd = torch.full((M, N), float("nan"), device="cuda")
        path = cabi.gemm(M, N, K, A.data_ptr(), a.shape[1], B.data_ptr(), b.shape[1], Cd.data_ptr(),
                         N, trans_a=ta, trans_b=tb, precision=1, workspace=ws.data_ptr(),
                         workspace_bytes=ws.numel())
        torch.cuda.synchronize()
        assert path == 1
        return Cd.cpu().numpy()

    cp, cs = _both(run)
    a64 = (a.T if ta else a).astype(np.float64)
    b64 = (b.T if tb else b).astype(np.float64)
    want = a64 @ b64
    tol = _tol(a64, b64)
    assert np.all(np.abs(cp - want) <= tol)
    assert np.all(np.abs(cs - want) <= tol)
    assert np.abs(cp - cs).max() <= tol.max()


@pytest.mark.parametrize("shape", [(1100, 2048, 512), (4100, 512, 2048), (2048, 4100, 600)])
def test_pair_epilogues(pair_modes, shape):
    """bias + ReLU + relu_mask_out; fused residual (addend); beta * C; float
    gate; gate bit mask -- pairs vs single tiles vs fp64."""
    import torch
    rng = np.random.default_rng(2)
    M, N, K = shape
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    r = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    gate = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    A, B, Bi, Rd, Gd = (torch.from_numpy(x).cuda() for x in (a, b, bias, r, gate))
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    mw = (N + 31) // 32
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    prod = a64 @ b64
    tol = _tol(a64, b64, 2.0)

    def gemm(Cd, **kw):
        path = cabi.gemm(M, N, K, A.data_ptr(), K, B.data_ptr(), N, Cd.data_ptr(), N, precision=1,
                         workspace=ws.data_ptr(), workspace_bytes=ws.numel(), **kw)
        torch.cuda.synchronize()
        assert path == 1

    # bias + ReLU + mask
    def relu_mask():
        Cd = torch.full((M, N), float("nan"), device="cuda")
        mask = torch.zeros(M * mw, dtype=torch.int32, device="cuda")
        gemm(Cd, bias=Bi.data_ptr(), relu=True, relu_mask_out=mask.data_ptr())
        return Cd.cpu().numpy(), mask.cpu().numpy().view(np.uint32).reshape(M, mw)

    (cp, mp), (cs, ms) = _both(relu_mask)
    want = np.maximum(prod + bias, 0)
    assert np.all(np.abs(cp - want) <= tol) and np.all(np.abs(cs - want) <= tol)
    for c, m in ((cp, mp), (cs, ms)):
        bits = np.zeros((M, mw * 32), bool)
        bits[:, :N] = c > 0
        packed = np.packbits(bits.reshape(M, mw, 4, 8)[..., ::-1], axis=-1).reshape(M, mw, 4)
        words = (packed[..., 0].astype(np.uint32) | packed[..., 1].astype(np.uint32) << 8 |
                 packed[..., 2].astype(np.uint32) << 16 | packed[..., 3].astype(np.uint32) << 24)
        assert np.array_equal(m, words)

    # fused residual: C = A B + bias + R (C write-only)
    def resid():
        Cd = torch.full((M, N), float("nan"), device="cuda")
        gemm(Cd, beta=1.0, bias=Bi.data_ptr(), addend=Rd.data_ptr())
        return Cd.cpu().numpy()

    cp, cs = _both(resid)
    want = prod + bias + r
    assert np.all(np.abs(cp - want) <= tol) and np.all(np.abs(cs - want) <= tol)

    # beta * C (accumulate into C)
    def beta_c():
        Cd = torch.from_numpy(r.copy()).cuda()
        gemm(Cd, beta=0.5)
        return Cd.cpu().numpy()

    cp, cs = _both(beta_c)
    want = prod + 0.5 * r
    assert np.all(np.abs(cp - want) <= tol) and np.all(np.abs(cs - want) <= tol)

    # float ReLU gate
    def gated():
        Cd = torch.full((M, N), float("nan"), device="cuda")
        gemm(Cd, gate=Gd.data_ptr())
        return Cd.cpu().numpy()

    cp, cs = _both(gated)
    want = np.where(gate > 0, prod, 0)
    assert np.all(np.abs(cp - want) <= tol) and np.all(np.abs(cs - want) <= tol)

    # gate as a bit mask (the FFN2 dX epilogue)
    gbits = np.zeros((M, mw * 32), bool)
    gbits[:, :N] = gate > 0
    gp = np.packbits(gbits.reshape(M, mw, 4, 8)[..., ::-1], axis=-1).reshape(M, mw, 4)
    gwords = (gp[..., 0].astype(np.uint32) | gp[..., 1].astype(np.uint32) << 8 |
              gp[..., 2].astype(np.uint32) << 16 | gp[..., 3].astype(np.uint32) << 24)
    Gm = torch.from_numpy(gwords.view(np.int32).copy()).cuda()

    def gated_mask():
        Cd = torch.full((M, N), float("nan"), device="cuda")
        gemm(Cd, gate_mask=Gm.data_ptr())
        return Cd.cpu().numpy()

    cp, cs = _both(gated_mask)
    assert np.all(np.abs(cp - want) <= tol) and np.all(np.abs(cs - want) <= tol)


@pytest.mark.parametrize("which", ["B", "A"])
@pytest.mark.parametrize("shape", [(2048, 512, 6500), (32000, 512, 1500), (1500, 2048, 7000)])
def test_pair_fused_colsum(pair_modes, which, shape):
    """dW = X^T dY with db = colsum(dY) fused (operand sums taken per CTA over
    its own staged half; the odd CTA relays its stage arrivals)."""
    import torch
    rng = np.random.default_rng(3)
    M, N, K = shape
    dy_cols = N if which == "B" else M
    x_cols = M if which == "B" else N
    dy = rng.uniform(-1, 1, (K, dy_cols)).astype(np.float32)
    x = rng.uniform(-1, 1, (K, x_cols)).astype(np.float32)
    Dy, X = torch.from_numpy(dy).cuda(), torch.from_numpy(x).cuda()
    A, B = (X, Dy) if which == "B" else (Dy, X)
    lda, ldb = (x_cols, dy_cols) if which == "B" else (dy_cols, x_cols)
    ws = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def run():
        cs = torch.full((dy_cols,), float("nan"), device="cuda")
        Cd = torch.full((M, N), float("nan"), device="cuda")
        path = cabi.gemm(M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, Cd.data_ptr(), N,
                         trans_a=True, precision=1, workspace=ws.data_ptr(),
                         workspace_bytes=ws.numel(), colsum=cs.data_ptr(),
                         colsum_of=2 if which == "B" else 1)
        torch.cuda.synchronize()
        assert path == 1
        return Cd.cpu().numpy(), cs.cpu().numpy()

    (cp, sp), (cs_, ss) = _both(run)
    want_s = dy.astype(np.float64).sum(0)
    stol = 2.0 ** -11 * np.abs(dy).astype(np.float64).sum(0) * 1.05 + 1e-5
    assert np.all(np.abs(sp - want_s) <= stol) and np.all(np.abs(ss - want_s) <= stol)
    a64 = x.T.astype(np.float64) if which == "B" else dy.T.astype(np.float64)
    b64 = dy.astype(np.float64) if which == "B" else x.astype(np.float64)
    want = a64 @ b64
    tol = _tol(a64, b64, 1.0)
    assert np.all(np.abs(cp - want) <= tol) and np.all(np.abs(cs_ - want) <= tol)


@pytest.mark.parametrize("shape", [(2100, 512, 512), (1024, 1000, 2048)])
def test_pair_group_and_kconcat(pair_modes, shape):
    """q/k/v-style groups (one A, three B) and the K-concatenated dX sum."""
    import torch
    rng = np.random.default_rng(4)
    M, N, K = shape
    As = [rng.uniform(-1, 1, (M, K)).astype(np.float32) for _ in range(3)]
    Bs = [rng.uniform(-1, 1, (K, N)).astype(np.float32) for _ in range(3)]
    bs = [rng.uniform(-1, 1, N).astype(np.float32) for _ in range(3)]
    dA = [torch.from_numpy(x).cuda() for x in As]
    dB = [torch.from_numpy(x).cuda() for x in Bs]
    db = [torch.from_numpy(x).cuda() for x in bs]
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def grouped():
        Cs = [torch.full((M, N), float("nan"), device="cuda") for _ in range(3)]
        cabi.gemm_group(M, N, K, [(dA[0].data_ptr(), dB[q].data_ptr(), Cs[q].data_ptr(),
                                   db[q].data_ptr()) for q in range(3)], K, N, N,
                        workspace=ws.data_ptr(), workspace_bytes=ws.numel())
        torch.cuda.synchronize()
        return [c.cpu().numpy() for c in Cs]

    gp, gs = _both(grouped)
    for q in range(3):
        a64, b64 = As[0].astype(np.float64), Bs[q].astype(np.float64)
        want = a64 @ b64 + bs[q]
        tol = _tol(a64, b64, 2.0)
        assert np.all(np.abs(gp[q] - want) <= tol) and np.all(np.abs(gs[q] - want) <= tol)

    c0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)

    def kcat():
        Cd = torch.from_numpy(c0.copy()).cuda()
        cabi.gemm_group(M, N, K, [(dA[q].data_ptr(), dB[q].data_ptr(), Cd.data_ptr(), None)
                                  for q in range(3)], K, N, N, beta=1.0, kconcat=True,
                        workspace=ws.data_ptr(), workspace_bytes=ws.numel())
        torch.cuda.synchronize()
        return Cd.cpu().numpy()

    kp, ks = _both(kcat)
    want = c0 + sum(As[q].astype(np.float64) @ Bs[q] for q in range(3))
    tol = sum(_tol(As[q].astype(np.float64), Bs[q].astype(np.float64)) for q in range(3)) + 1e-5
    assert np.all(np.abs(kp - want) <= tol) and np.all(np.abs(ks - want) <= tol)


def test_pair_switch_exported(cuda):
    L = cabi.lib()
    assert L.mtkc_gemm_set_pair(C.c_int(0)) == 0
    assert L.mtkc_gemm_set_pair(C.c_int(1)) == 0
