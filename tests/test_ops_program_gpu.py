"""Op-level parity for the elementwise / broadcast (a4), reduce (a5) and
layout (a6) rows against the unmodified reference, through the public graph
API on both sides.

Each case is a small stack program of graph ops (same grammar as
oracle/ref_shim.cpp `ref_op_program`): the reference runs it on its
ExpressionGraph, this build runs it on the B200 graph, both with the loss
sum(out * G), and the output and every input gradient are compared.

Reference: src/graph.cpp:139-268 (binary/unary + reduce-to-shape backward),
:338-459 (reshape/transpose/concat/slice/gatherRows), :463-524 (reduce,
argmax ties -> lowest index), src/tensor.cpp:160-237, 322-368, 480-541;
KATs tests/test_tensor.cpp:79-139.

Tolerances: layout ops, add/sub/neg/scale/relu, max/argmax and their
backward are exact data movement or single roundings in the reference order
-> bit-exact.  mul/div, sums and means re-associated across threads and
transcendental functions (CUDA vs glibc exp/tanh/log, ulp-level) -> 2e-6
relative to the output scale.
"""
import zlib

import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import mtk as M

pytestmark = pytest.mark.gpu

RED = {"sum": "Sum", "max": "Max", "mean": "Mean", "argmax": "Argmax"}


def run_mine(prog, inputs, G):
    g = M.ExpressionGraph(1)
    params = [g.param(f"p{i}", list(a.shape), np.ascontiguousarray(a, np.float32))
              for i, a in enumerate(inputs)]
    st = []
    for tok in prog.split():
        f = tok.split(":")
        op = f[0]
        if op[0] == "p" and op[1:].isdigit():
            st.append(params[int(op[1:])])
        elif op == "dup":
            st.append(st[-1])
        elif op in ("add", "sub", "mul", "div"):
            b, a = st.pop(), st.pop()
            st.append(getattr(g, op)(a, b))
        elif op in ("tanh", "sigmoid", "relu", "exp", "log", "neg"):
            st.append(getattr(g, op)(st.pop()))
        elif op == "scale":
            st.append(g.scale(st.pop(), float(f[1])))
        elif op == "adds":
            st.append(g.add_scalar(st.pop(), float(f[1])))
        elif op == "reshape":
            st.append(g.reshape(st.pop(), [int(x) for x in f[1].split(",")]))
        elif op == "transpose":
            st.append(g.transpose(st.pop(), [int(x) for x in f[1].split(",")]))
        elif op == "concat":
            n, axis = int(f[1]), int(f[2])
            parts = st[-n:]
            del st[-n:]
            st.append(g.concat(parts, axis))
        elif op == "slice":
            st.append(g.slice(st.pop(), int(f[1]), int(f[2]), int(f[3])))
        elif op == "gather":
            st.append(g.gather_rows(st.pop(), [int(x) for x in f[1].split(",")]))
        elif op == "reduce":
            st.append(g.reduce(getattr(M.ReduceOp, RED[f[1]]), st.pop(), int(f[2]), bool(int(f[3]))))
        elif op == "softmax":
            st.append(g.softmax(st.pop(), None))
        else:
            raise ValueError(tok)
    out = st.pop()
    shape = tuple(out.shape)
    Gf = np.asarray(G, np.float32).reshape(shape)
    n = int(np.prod(shape))
    loss = g.reduce(M.ReduceOp.Sum, g.reshape(g.mul(out, g.constant(Gf)), [1, n]), 1)
    g.forward()
    g.zero_grads()
    g.backward(loss)
    return out.val().reshape(shape), [g.param_grad(f"p{i}") for i in range(len(inputs))]


def out_shape(prog, inputs):
    """Output shape from the reference (G of ones is only used for its size)."""
    big = np.ones(1 << 16, np.float32)
    out, _ = R.op_program(prog, inputs, big)
    return out.shape


U = lambda rng, *s: rng.uniform(-1, 1, s).astype(np.float32)  # noqa: E731
P = lambda rng, *s: rng.uniform(0.5, 2, s).astype(np.float32)  # noqa: E731

# (id, program, input factory, exact?)
CASES = [
    ("add_same", "p0 p1 add", lambda r: [U(r, 3, 5), U(r, 3, 5)], True),
    ("add_bcast_row", "p0 p1 add", lambda r: [U(r, 4, 6), U(r, 6)], True),
    ("add_bcast_col", "p0 p1 add", lambda r: [U(r, 2, 4, 6), U(r, 4, 1)], True),
    ("add_bcast_left", "p0 p1 add", lambda r: [U(r, 6), U(r, 3, 6)], True),
    ("sub_bcast", "p0 p1 sub", lambda r: [U(r, 2, 3, 4), U(r, 1, 3, 4)], True),
    ("mul_bcast", "p0 p1 mul", lambda r: [U(r, 5, 7), U(r, 7)], False),
    ("div_bcast", "p0 p1 div", lambda r: [U(r, 4, 6), P(r, 6)], False),
    ("self_add", "p0 tanh dup add", lambda r: [U(r, 3, 8)], False),
    ("self_add_reshape", "p0 tanh dup reshape:24 add", lambda r: [U(r, 24)], False),
    ("self_mul", "p0 sigmoid dup mul", lambda r: [U(r, 4, 4)], False),
    ("tanh", "p0 tanh", lambda r: [U(r, 7, 9)], False),
    ("sigmoid", "p0 sigmoid", lambda r: [U(r, 7, 9)], False),
    ("relu", "p0 relu", lambda r: [U(r, 7, 9)], True),
    ("exp", "p0 exp", lambda r: [U(r, 7, 9)], False),
    ("log", "p0 log", lambda r: [P(r, 7, 9)], False),
    ("neg", "p0 neg", lambda r: [U(r, 7, 9)], True),
    ("scale", "p0 scale:0.125", lambda r: [U(r, 5, 3)], True),
    ("add_scalar", "p0 adds:1.5", lambda r: [U(r, 5, 3)], True),
    ("reduce_sum_last", "p0 reduce:sum:1:0", lambda r: [U(r, 6, 33)], False),
    ("reduce_sum_first_keep", "p0 reduce:sum:0:1", lambda r: [U(r, 6, 33)], False),
    ("reduce_mean_mid", "p0 reduce:mean:1:0", lambda r: [U(r, 3, 5, 7)], False),
    ("reduce_max", "p0 reduce:max:1:0", lambda r: [U(r, 5, 17)], True),
    ("reduce_max_ties", "p0 reduce:max:1:1",
     lambda r: [np.array([[1, 3, 3, 0], [2, 2, 2, 2], [-1, -1, -5, -1]], np.float32)], True),
    ("argmax_ties", "p0 reduce:argmax:1:0",
     lambda r: [np.array([[1, 3, 3, 0], [2, 2, 2, 2], [-1, -1, -5, -1]], np.float32)], True),
    ("transpose_2d", "p0 transpose:1,0", lambda r: [U(r, 5, 9)], True),
    ("transpose_heads", "p0 transpose:0,2,1,3", lambda r: [U(r, 2, 5, 4, 3)], True),
    ("transpose_3d", "p0 transpose:2,0,1", lambda r: [U(r, 3, 4, 5)], True),
    ("reshape_chain", "p0 reshape:6,4 transpose:1,0 reshape:24", lambda r: [U(r, 2, 3, 4)], True),
    ("concat_last", "p0 p1 concat:2:1", lambda r: [U(r, 4, 3), U(r, 4, 5)], True),
    ("concat_first", "p0 p1 p2 concat:3:0", lambda r: [U(r, 1, 6), U(r, 2, 6), U(r, 3, 6)], True),
    ("concat_mid", "p0 p1 concat:2:1", lambda r: [U(r, 2, 3, 4), U(r, 2, 1, 4)], True),
    ("slice_last", "p0 slice:1:2:3", lambda r: [U(r, 4, 8)], True),
    ("slice_time", "p0 slice:1:1:1", lambda r: [U(r, 3, 5, 4)], True),
    ("gather_rows", "p0 gather:2,0,2,1", lambda r: [U(r, 3, 5)], True),
    ("gather_rows_dup_sum", "p0 gather:1,1,1,0", lambda r: [U(r, 2, 5)], True),
    ("softmax_plain", "p0 softmax", lambda r: [U(r, 4, 9)], False),
    ("composite", "p0 p1 mul p2 add tanh reduce:mean:0:0",
     lambda r: [U(r, 6, 4), U(r, 4), U(r, 6, 4)], False),
]


@pytest.fixture(autouse=True)
def fp32_mode(cuda):
    M.set_precision("fp32")
    yield
    M.set_precision("tf32")


@pytest.mark.parametrize("cid,prog,make,exact", CASES, ids=[c[0] for c in CASES])
def test_op_program_vs_reference(cid, prog, make, exact):
    rng = np.random.default_rng(zlib.crc32(cid.encode()))
    inputs = make(rng)
    shape = out_shape(prog, inputs)
    G = rng.uniform(-1, 1, shape).astype(np.float32)
    ro, rg = R.op_program(prog, inputs, G)
    mo, mg = run_mine(prog, inputs, G)
    assert mo.shape == ro.shape
    if exact:
        assert np.array_equal(mo, ro), np.abs(mo - ro).max()
        for a, b in zip(mg, rg):
            assert np.array_equal(a.reshape(b.shape), b), np.abs(a.reshape(b.shape) - b).max()
    else:
        tol = 2e-6
        scale = max(float(np.abs(ro).max()), 1e-30)
        assert np.abs(mo - ro).max() <= tol * scale, np.abs(mo - ro).max() / scale
        for a, b in zip(mg, rg):
            s = max(float(np.abs(b).max()), 1e-30)
            assert np.abs(a.reshape(b.shape) - b).max() <= tol * s, np.abs(a.reshape(b.shape) - b).max() / s


def test_self_add_gradient_doubles():
    """add(h, h) with h = tanh(x), not a parameter: dh = 2 go, so
    dx = 2 (1 - tanh^2 x) (graph.cpp:155-176 accumulate both operands)."""
    x = np.linspace(-1, 1, 12, dtype=np.float32).reshape(3, 4)
    _, (gx,) = run_mine("p0 tanh dup add", [x], np.ones((3, 4), np.float32))
    np.testing.assert_allclose(gx, 2 * (1 - np.tanh(x.astype(np.float64)) ** 2), rtol=1e-6, atol=1e-6)


def test_division_by_zero_is_numeric_error():
    """ewiseBinaryInto Div throws NumericError on a zero divisor
    (tensor.cpp:161-165); the reference raises the same type."""
    a = np.ones((2, 3), np.float32)
    b = np.array([1, 0, 2], np.float32)
    with pytest.raises(R.RefError, match="NumericError"):
        R.op_program("p0 p1 div", [a, b], np.ones((2, 3), np.float32))
    g = M.ExpressionGraph(1)
    pa = g.param("a", [2, 3], a)
    pb = g.param("b", [3], b)
    g.div(pa, pb)
    with pytest.raises(M.NumericError):
        g.forward()
        M.check_flags()
    M.sync()


def test_device_error_step_does_not_update_parameters():
    """A step whose forward raised a device error (division by zero,
    tensor.cpp:161-165) throws NumericError at the update and -- as in the
    reference, which throws inside forward before Adam (train.cpp:226-272) --
    leaves every parameter and the step counter untouched: the device error
    word joins the optimizer's skip flag (mtkc_flag_or)."""
    g = M.ExpressionGraph(1)
    pa = g.param("a", [2, 3], np.ones((2, 3), np.float32))
    pb = g.param("b", [3], np.array([1, 0, 2], np.float32))
    before = {n: g.param_value(n).copy() for n in ("a", "b")}
    out = g.div(pa, pb)
    loss = g.reduce(M.ReduceOp.Sum, g.reshape(out, [1, 6]), 1)
    g.forward()
    g.zero_grads()
    g.backward(loss)
    adam = M.Adam(M.AdamConfig())
    with pytest.raises(M.NumericError, match="division by zero"):
        adam.update(g, 1e-2)
    for n in before:
        assert np.array_equal(g.param_value(n), before[n]), n
    assert adam.step() == 0
    M.check_flags()  # the error was consumed: later steps start clean
