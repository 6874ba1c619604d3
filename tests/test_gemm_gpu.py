"""GEMM parity: the C-ABI mtkc_gemm against the reference's matmulInto
(tensor.cpp:258-306) run from oracle/_ref, for every transpose case.

* FP32 (CUDA-core) path: bit-exact with the reference (same summation order,
  separately rounded multiply/add).
* TF32 tcgen05 path: |C - C64| <= 4e-3 * (|A||B|)_ij  (tf32 has a 10-bit
  mantissa; the bound is on the absolute-value product, so it holds for any
  cancellation pattern).
"""
import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import cabi

pytestmark = pytest.mark.gpu


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _run(torch, a, b, ta, tb, alpha=1.0, beta=0.0, c0=None, precision=0, bias=None, relu=False,
         gate=None):
    M = a.shape[1] if ta else a.shape[0]
    K = a.shape[0] if ta else a.shape[1]
    N = b.shape[0] if tb else b.shape[1]
    A, B = _dev(torch, a), _dev(torch, b)
    Cd = _dev(torch, c0 if c0 is not None else np.zeros((M, N), np.float32))
    bd = _dev(torch, bias) if bias is not None else None
    gd = _dev(torch, gate) if gate is not None else None
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    path = cabi.gemm(M, N, K, A.data_ptr(), a.shape[1], B.data_ptr(), b.shape[1], Cd.data_ptr(), N,
                     trans_a=ta, trans_b=tb, alpha=alpha, beta=beta,
                     bias=bd.data_ptr() if bd is not None else None, relu=relu,
                     gate=gd.data_ptr() if gd is not None else None,
                     precision=precision, workspace=ws.data_ptr(), workspace_bytes=ws.numel())
    torch.cuda.synchronize()
    return Cd.cpu().numpy(), path


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("shape", [(7, 5, 3), (64, 48, 80), (130, 70, 33)])
def test_fp32_gemm_bitexact_vs_reference(cuda, ta, tb, shape):
    import torch
    rng = np.random.default_rng(1)
    M, K, N = shape
    a = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
    c0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    for alpha, beta in [(1.0, 0.0), (1.0, 1.0), (0.5, 2.0)]:
        ref = R.matmul(a, b, bool(ta), bool(tb), alpha, beta, c0)
        got, path = _run(torch, a, b, ta, tb, alpha, beta, c0, precision=0)
        assert path == 0
        assert np.array_equal(got, ref), f"max diff {np.abs(got - ref).max()}"


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("shape", [(128, 64, 128), (256, 512, 384), (300, 520, 200),
                                   (1024, 4096, 512), (512, 8192, 512)])
def test_tf32_tcgen05_gemm(cuda, ta, tb, shape):
    import torch
    rng = np.random.default_rng(2)
    M, K, N = shape
    a = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
    opa = a.T if ta else a
    opb = b.T if tb else b
    exact = opa.astype(np.float64) @ opb.astype(np.float64)
    bound = np.abs(opa).astype(np.float64) @ np.abs(opb).astype(np.float64)
    got, path = _run(torch, a, b, ta, tb, precision=1)
    assert path == 1, "tensor-core path not taken"
    err = np.abs(got - exact)
    assert np.all(err <= 4e-3 * bound + 1e-6), f"max rel {np.max(err / (bound + 1e-9))}"


def test_tf32_epilogues(cuda):
    import torch
    rng = np.random.default_rng(3)
    M, K, N = 256, 256, 384
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    c0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    exact = a.astype(np.float64) @ b.astype(np.float64)
    bound = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64) + 1
    got, _ = _run(torch, a, b, 0, 0, precision=1, bias=bias, relu=True)
    want = np.maximum(exact + bias, 0)
    assert np.all(np.abs(got - want) <= 4e-3 * bound)
    got, _ = _run(torch, a, b, 0, 0, alpha=0.5, beta=1.0, c0=c0, precision=1)
    want = 0.5 * exact + c0
    assert np.all(np.abs(got - want) <= 4e-3 * bound)


@pytest.mark.parametrize("shape", [(256, 256, 384), (200, 96, 300), (70, 8192, 96), (333, 64, 2050)])
def test_tf32_epilogue_combinations(cuda, shape):
    """bias (vector and ragged), ReLU gate (TMA-loaded box), beta*C (TMA-loaded
    box), gate+beta together, and the split-K reduction (long K)."""
    import torch
    rng = np.random.default_rng(4)
    M, K, N = shape
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    c0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    gate = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    exact = a.astype(np.float64) @ b.astype(np.float64)
    tol = 4e-3 * (np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64) + 1)
    cases = [
        (dict(bias=bias), exact + bias),
        (dict(bias=bias, relu=True), np.maximum(exact + bias, 0)),
        (dict(gate=gate), np.where(gate > 0, exact, 0)),
        (dict(beta=1.0, c0=c0), exact + c0),
        (dict(beta=2.0, c0=c0, gate=gate, alpha=0.5), 2.0 * c0 + np.where(gate > 0, 0.5 * exact, 0)),
    ]
    for kw, want in cases:
        got, path = _run(torch, a, b, 0, 0, precision=1, **kw)
        assert path == 1 or N % 4, "tensor-core path not taken"  # TMA needs 16-B row pitch
        err = np.abs(got - want)
        assert np.all(err <= tol), (kw.keys(), float(np.max(err - tol)))


@pytest.mark.parametrize("shape", [(300, 128, 256), (1000, 512, 512), (64, 8192, 96), (517, 40, 2050)])
def test_tf32_gemm_group(cuda, shape):
    """mtkc_gemm_group: three products of one shape in one launch -- independent
    outputs with per-problem bias (q/k/v forward), the K-concatenated sum into
    one output with beta (their dX), and transposed-A products with split-K
    (their dW)."""
    import torch
    rng = np.random.default_rng(5)
    M, K, N = shape
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    As = [rng.uniform(-1, 1, (M, K)).astype(np.float32) for _ in range(3)]
    Bs = [rng.uniform(-1, 1, (K, N)).astype(np.float32) for _ in range(3)]
    bs = [rng.uniform(-1, 1, N).astype(np.float32) for _ in range(3)]
    dA, dB, db = [dev(x) for x in As], [dev(x) for x in Bs], [dev(x) for x in bs]
    tol = lambda a, b: 4e-3 * (np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64) + 1)
    # independent outputs sharing A (forward of q/k/v)
    Cs = [torch.zeros(M, N, device="cuda") for _ in range(3)]
    path = cabi.gemm_group(M, N, K, [(dA[0].data_ptr(), dB[q].data_ptr(), Cs[q].data_ptr(),
                                     db[q].data_ptr()) for q in range(3)], K, N, N,
                           workspace=ws.data_ptr(), workspace_bytes=ws.numel())
    torch.cuda.synchronize()
    assert path == 1 or N % 4
    for q in range(3):
        want = As[0].astype(np.float64) @ Bs[q] + bs[q]
        assert np.all(np.abs(Cs[q].cpu().numpy() - want) <= tol(As[0], Bs[q])), q
    # K-concatenated sum with beta = 1 (dX = sum_q dY_q W_q^T)
    c0 = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    Cd = dev(c0)
    cabi.gemm_group(M, N, K, [(dA[q].data_ptr(), dB[q].data_ptr(), Cd.data_ptr(), None)
                              for q in range(3)], K, N, N, beta=1.0, kconcat=True,
                    workspace=ws.data_ptr(), workspace_bytes=ws.numel())
    torch.cuda.synchronize()
    want = c0 + sum(As[q].astype(np.float64) @ Bs[q] for q in range(3))
    bound = sum(tol(As[q], Bs[q]) for q in range(3))
    assert np.all(np.abs(Cd.cpu().numpy() - want) <= bound)
    # transposed A shared, long contraction (dW_q = X^T dY_q), beta = 0
    Xt = [dev(x) for x in As]  # storage [M x K] read as op(A) = A^T  -> [K x M] @ [M x N]
    Ys = [dev(rng.uniform(-1, 1, (M, N)).astype(np.float32)) for _ in range(3)]
    Ws = [torch.zeros(K, N, device="cuda") for _ in range(3)]
    cabi.gemm_group(K, N, M, [(Xt[0].data_ptr(), Ys[q].data_ptr(), Ws[q].data_ptr(), None)
                              for q in range(3)], K, N, N, trans_a=True,
                    workspace=ws.data_ptr(), workspace_bytes=ws.numel())
    torch.cuda.synchronize()
    for q in range(3):
        y = Ys[q].cpu().numpy()
        want = As[0].T.astype(np.float64) @ y
        assert np.all(np.abs(Ws[q].cpu().numpy() - want) <= tol(As[0].T, y)), q


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("shape", [(300, 256, 512), (70, 8192, 96), (33, 40, 50)])
def test_gemm_addend(cuda, prec, shape):
    """Fused residual: C = A B + bias + beta * R with R a separate tensor
    (mtkc_gemm_args.addend); C is write-only.  FP32 and TF32 paths, incl. the
    split-K reduction (long K) and ragged shapes."""
    import torch
    rng = np.random.default_rng(7)
    M, K, N = shape
    a = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    r = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    A, B, Bi, Rd = (torch.from_numpy(x).cuda() for x in (a, b, bias, r))
    Cd = torch.full((M, N), float("nan"), device="cuda")
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    cabi.gemm(M, N, K, A.data_ptr(), K, B.data_ptr(), N, Cd.data_ptr(), N, beta=1.0,
              bias=Bi.data_ptr(), addend=Rd.data_ptr(), precision=prec,
              workspace=ws.data_ptr(), workspace_bytes=ws.numel())
    torch.cuda.synchronize()
    want = a.astype(np.float64) @ b + bias + r
    tol = 4e-3 * (np.abs(a).astype(np.float64) @ np.abs(b) + 2)
    got = Cd.cpu().numpy()
    assert np.all(np.isfinite(got))
    assert np.all(np.abs(got - want) <= tol)
    assert torch.equal(Rd.cpu(), torch.from_numpy(r))  # addend untouched


def _colsum_direct(torch, x, out, acc, ws):
    import ctypes as C
    rows, cols = x.shape
    cabi.check(cabi.lib().mtkc_colsum(C.c_void_p(out.data_ptr()), C.c_void_p(x.data_ptr()),
                                      C.c_int64(rows), C.c_int64(cols), C.c_int(int(acc)),
                                      C.c_void_p(ws.data_ptr()), C.c_size_t(ws.numel()), None))


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("which", ["B", "A"])
@pytest.mark.parametrize("shape", [(512, 512, 8184), (96, 40, 300), (256, 520, 1000),
                                   (2048, 512, 4096)])
def test_gemm_fused_colsum(cuda, prec, which, shape):
    """mtkc_gemm_args.colsum: the bias gradient db = colsum(dY) produced by the
    dW product itself.  which = "B": dW = X^T dY (colsum of op(B) = dY);
    "A": dW = dY^T X (the tied output layer; row sums of op(A) = dY^T).
    Both with and without split-K, fresh and accumulating.  FP32 precision:
    bit-identical to mtkc_colsum; TF32: the sums of the tf32-rounded operand,
    |db - db64| <= 2^-11 sum|dY| (+ fp32 accumulation)."""
    import torch
    rng = np.random.default_rng(11)
    M, N, K = shape  # op(A) M x K, op(B) K x N ; K = token rows
    dy_cols = N if which == "B" else M
    x_cols = M if which == "B" else N
    dy = rng.uniform(-1, 1, (K, dy_cols)).astype(np.float32)
    x = rng.uniform(-1, 1, (K, x_cols)).astype(np.float32)
    Dy, X = _dev(torch, dy), _dev(torch, x)
    A, B = (X, Dy) if which == "B" else (Dy, X)
    lda, ldb = (x_cols, dy_cols) if which == "B" else (dy_cols, x_cols)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    ws2 = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    want = dy.astype(np.float64).sum(0)
    for acc in (False, True):
        cs0 = rng.uniform(-1, 1, dy_cols).astype(np.float32)
        cs = _dev(torch, cs0) if acc else torch.full((dy_cols,), float("nan"), device="cuda")
        Cd = torch.zeros(M, N, device="cuda")
        cabi.gemm(M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, Cd.data_ptr(), N, trans_a=True,
                  precision=prec, workspace=ws.data_ptr(), workspace_bytes=ws.numel(),
                  colsum=cs.data_ptr(), colsum_of=2 if which == "B" else 1,
                  colsum_accumulate=acc)
        torch.cuda.synchronize()
        got = cs.cpu().numpy()
        if prec == 0:
            ref = _dev(torch, cs0) if acc else torch.zeros(dy_cols, device="cuda")
            _colsum_direct(torch, Dy, ref, acc, ws2)
            torch.cuda.synchronize()
            assert np.array_equal(got, ref.cpu().numpy())
        else:
            base = cs0.astype(np.float64) if acc else 0.0
            tol = 2.0 ** -11 * np.abs(dy).astype(np.float64).sum(0) * 1.05 + 1e-5 * (1 + np.abs(base))
            assert np.all(np.abs(got - (base + want)) <= tol), float(np.max(np.abs(got - base - want) - tol))
        if acc:  # the product itself is unaffected by the fused sums
            a64 = x.T.astype(np.float64) if which == "B" else dy.T.astype(np.float64)
            b64 = dy.astype(np.float64) if which == "B" else x.astype(np.float64)
            c = Cd.cpu().numpy()
            assert np.all(np.abs(c - a64 @ b64) <= 4e-3 * (np.abs(a64) @ np.abs(b64) + 1))


def test_gemm_group_fused_colsum(cuda):
    """Grouped dW_q = X^T dY_q with db_q = colsum(dY_q) in the same launch."""
    import torch
    rng = np.random.default_rng(12)
    rows, K, N = 8184, 512, 512
    x = rng.uniform(-1, 1, (rows, K)).astype(np.float32)
    dys = [rng.uniform(-1, 1, (rows, N)).astype(np.float32) for _ in range(3)]
    X, Dy = _dev(torch, x), [_dev(torch, d) for d in dys]
    Ws = [torch.zeros(K, N, device="cuda") for _ in range(3)]
    cs = [torch.full((N,), float("nan"), device="cuda") for _ in range(3)]
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    path = cabi.gemm_group(K, N, rows, [(X.data_ptr(), Dy[q].data_ptr(), Ws[q].data_ptr(), None,
                                         cs[q].data_ptr()) for q in range(3)], K, N, N,
                           trans_a=True, workspace=ws.data_ptr(), workspace_bytes=ws.numel(),
                           colsum_of=2)
    torch.cuda.synchronize()
    assert path == 1
    for q in range(3):
        want = dys[q].astype(np.float64).sum(0)
        tol = 2.0 ** -11 * np.abs(dys[q]).astype(np.float64).sum(0) * 1.05 + 1e-5
        assert np.all(np.abs(cs[q].cpu().numpy() - want) <= tol), q
        w = x.T.astype(np.float64) @ dys[q]
        assert np.all(np.abs(Ws[q].cpu().numpy() - w) <= 4e-3 * (np.abs(x.T) @ np.abs(dys[q]) + 1)), q


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("shape", [(300, 70, 96), (1000, 2048, 512), (64, 2048, 8192)])
def test_gemm_relu_bitmask(cuda, prec, shape):
    """relu_mask_out / gate_mask: the ReLU producer's gate packed to one bit per
    element (word [r][c/32], bits past N zero), and a consumer gated by it
    equals the same consumer gated by the float ReLU output (bitwise) --
    direct epilogue, split-K reduction (long K) and the CUDA-core path."""
    import torch
    rng = np.random.default_rng(13)
    M, N, K = shape
    mw = (N + 31) // 32
    a = _dev(torch, rng.uniform(-1, 1, (M, 64)))
    b = _dev(torch, rng.uniform(-1, 1, (64, N)))
    bias = _dev(torch, rng.uniform(-0.5, 0.5, N))
    h = torch.zeros(M, N, device="cuda")
    mask = torch.full((M, mw), -1, dtype=torch.int32, device="cuda")
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    cabi.gemm(M, N, 64, a.data_ptr(), 64, b.data_ptr(), N, h.data_ptr(), N, bias=bias.data_ptr(),
              relu=True, precision=prec, workspace=ws.data_ptr(), workspace_bytes=ws.numel(),
              relu_mask_out=mask.data_ptr())
    torch.cuda.synchronize()
    hv = h.cpu().numpy()
    words = mask.cpu().numpy().view(np.uint32)
    bits = (words[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1
    bits = bits.reshape(M, mw * 32)
    assert np.array_equal(bits[:, :N] == 1, hv > 0)
    assert not bits[:, N:].any()
    # consumer: dH = dY W^T gated, K = the consumer's contraction
    dy = _dev(torch, rng.uniform(-1, 1, (M, K)))
    w = _dev(torch, rng.uniform(-1, 1, (N, K)))
    outs = []
    for use_mask in (False, True):
        o = torch.zeros(M, N, device="cuda")
        cabi.gemm(M, N, K, dy.data_ptr(), K, w.data_ptr(), K, o.data_ptr(), N, trans_b=True,
                  gate=None if use_mask else h.data_ptr(),
                  gate_mask=mask.data_ptr() if use_mask else None, precision=prec,
                  workspace=ws.data_ptr(), workspace_bytes=ws.numel())
        torch.cuda.synchronize()
        outs.append(o.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    assert np.all(outs[1][hv <= 0] == 0)
