"""ctypes view of the C-ABI kernel seam, libmtkcuda.so (include/mtk_cuda.h).

This is the binding a foreign host (cgo / JNI / Python) would write against
the drop-in boundary; the tests use it to call single kernels on device
buffers.  Loading fails loudly when the library is missing: there is no CPU
fallback anywhere on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmtkcuda.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "mtk_cuda.h")

_lib = None


class GemmArgs(C.Structure):
    _fields_ = [
        ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64), ("batch", C.c_int64),
        ("A", C.c_void_p), ("lda", C.c_int64), ("strideA", C.c_int64), ("transA", C.c_int),
        ("B", C.c_void_p), ("ldb", C.c_int64), ("strideB", C.c_int64), ("transB", C.c_int),
        ("C", C.c_void_p), ("ldc", C.c_int64), ("strideC", C.c_int64),
        ("alpha", C.c_float), ("beta", C.c_float),
        ("bias", C.c_void_p), ("epilogue", C.c_int), ("gate", C.c_void_p),
        ("precision", C.c_int), ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
        ("addend", C.c_void_p),
        ("colsum", C.c_void_p), ("colsum_of", C.c_int), ("colsum_accumulate", C.c_int),
        ("relu_mask_out", C.c_void_p), ("gate_mask", C.c_void_p),
    ]


def declared_symbols() -> list[str]:
    """Every function the public header declares."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|uint64_t|size_t)\s+(mtkc_\w+)\s*\(", text, re.M)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build with __graft_entry__.build() "
                               "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        L.mtkc_last_error.restype = C.c_char_p
        L.mtkc_launch_count.restype = C.c_uint64
        L.mtkc_gemm.argtypes = [C.POINTER(GemmArgs), C.c_void_p]
        L.mtkc_gemm_group.argtypes = [C.POINTER(GemmArgs), C.c_int, C.c_int, C.c_void_p]
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        raise RuntimeError(f"mtkc error {rc}: {lib().mtkc_last_error().decode()}")


def gemm(M, N, K, A, lda, B, ldb, Cp, ldc, trans_a=False, trans_b=False, alpha=1.0, beta=0.0,
         bias=None, relu=False, gate=None, precision=1, workspace=None, workspace_bytes=0,
         stream=None, batch=1, stride_a=0, stride_b=0, stride_c=0, addend=None, colsum=None,
         colsum_of=0, colsum_accumulate=False, relu_mask_out=None, gate_mask=None):
    g = GemmArgs(M, N, K, batch, A, lda, stride_a, int(trans_a), B, ldb, stride_b, int(trans_b),
                 Cp, ldc, stride_c, alpha, beta, bias, 1 if relu else 0, gate, precision,
                 workspace, workspace_bytes, addend, colsum, colsum_of, int(colsum_accumulate),
                 relu_mask_out, gate_mask)
    check(lib().mtkc_gemm(C.byref(g), stream))
    return lib().mtkc_gemm_last_path()


def gemm_group(M, N, K, probs, lda, ldb, ldc, trans_a=False, trans_b=False, alpha=1.0, beta=0.0,
               kconcat=False, precision=1, workspace=None, workspace_bytes=0, stream=None,
               colsum_of=0, colsum_accumulate=False):
    """mtkc_gemm_group: probs = [(A, B, C, bias-or-None[, colsum-or-None]), ...] device
    pointers."""
    arr = (GemmArgs * len(probs))()
    for i, pr in enumerate(probs):
        A, B, Cp, bias = pr[:4]
        cs = pr[4] if len(pr) > 4 else None
        arr[i] = GemmArgs(M, N, K, 1, A, lda, 0, int(trans_a), B, ldb, 0, int(trans_b), Cp, ldc, 0,
                          alpha, beta, bias, 0, None, precision, workspace, workspace_bytes, None,
                          cs, colsum_of if cs else 0, int(colsum_accumulate))
    check(lib().mtkc_gemm_group(arr, len(probs), int(kconcat), stream))
    return lib().mtkc_gemm_last_path()


def i64x4(dims):
    d = [1] * (4 - len(dims)) + list(dims)
    return (C.c_int64 * 4)(*d)
