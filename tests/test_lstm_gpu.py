"""Fused LSTM cell (north_star "fused GRU/LSTM cell ops"; kernels/lstm.cu).

The reference has no LSTM (gap 1), so the fused cell is
pinned the way the reference pins its own fused GRU (tests/gradsuite.h:304-
320: fused == unfused composition): the same cell written as a program of
the UNMODIFIED reference's graph primitives (dot, add, slice, sigmoid, tanh,
mul, concat on oracle/_ref's ExpressionGraph), same inputs, loss
sum(out * G).  Output and all six input gradients are compared: FP32 mode
(GEMMs in the reference's summation order) to 2e-6 of the output scale,
TF32 mode to 1e-2 per tensor.  Also: a two-step unrolled recurrence through
lstm_state / lstm_cell_state.
"""
import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import mtk as M

pytestmark = pytest.mark.gpu

B, IN, D = 24, 48, 64


def ref_program(d):
    pre = "p0 p3 dot p1 p4 dot add p5 add"  # h*U + x*W order does not matter here
    gate = lambda k, fn: f"{pre} slice:1:{k * d}:{d} {fn}"  # noqa: E731
    # c' = f*c + i*g ; out = [c' | h'] with h' = o*tanh(c')
    return (f"{gate(1, 'sigmoid')} p2 mul {gate(0, 'sigmoid')} {gate(3, 'tanh')} mul add "
            f"dup tanh {gate(2, 'sigmoid')} mul concat:2:1")


def inputs(seed):
    r = np.random.default_rng(seed)
    u = lambda *s: r.uniform(-1, 1, s).astype(np.float32)  # noqa: E731
    return [u(B, IN), u(B, D), u(B, D), u(IN, 4 * D) * 0.3, u(D, 4 * D) * 0.3, u(4 * D) * 0.5]


def mine(ins, G):
    g = M.ExpressionGraph(1)
    ps = [g.param(f"p{i}", list(a.shape), np.ascontiguousarray(a)) for i, a in enumerate(ins)]
    out = g.lstm_cell(*ps)  # [h' | c']
    loss = g.reduce(M.ReduceOp.Sum, g.reshape(g.mul(out, g.constant(G)), [1, B * 2 * D]), 1)
    g.forward()
    g.zero_grads()
    g.backward(loss)
    return out.val().reshape(B, 2 * D), [g.param_grad(f"p{i}").reshape(a.shape)
                                         for i, a in enumerate(ins)]


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_lstm_cell_vs_reference_composition(cuda, prec):
    ins = inputs(5)
    rng = np.random.default_rng(6)
    G = rng.uniform(-1, 1, (B, 2 * D)).astype(np.float32)
    Gref = np.concatenate([G[:, D:], G[:, :D]], axis=1)  # reference order [c' | h']
    ro, rg = R.op_program(ref_program(D), ins, Gref)
    ro = np.concatenate([ro[:, D:], ro[:, :D]], axis=1)
    M.set_precision(prec)
    try:
        mo, mg = mine(ins, G)
    finally:
        M.set_precision("tf32")
    if prec == "fp32":
        assert np.abs(mo - ro).max() <= 2e-6 * np.abs(ro).max()
        for a, b in zip(mg, rg):
            assert np.abs(a - b).max() <= 2e-6 * np.abs(b).max(), np.abs(a - b).max()
    else:
        assert np.linalg.norm(mo - ro) <= 1e-2 * np.linalg.norm(ro)
        for a, b in zip(mg, rg):
            assert np.linalg.norm(a - b) <= 1e-2 * np.linalg.norm(b), np.linalg.norm(a - b)


def test_lstm_two_step_recurrence(cuda):
    """h, c of step 1 feed step 2 (shared W, U, b): gradients flow through
    lstm_state / lstm_cell_state; compared with the same unrolled program on
    the reference."""
    ins = inputs(9)
    x2 = np.random.default_rng(10).uniform(-1, 1, (B, IN)).astype(np.float32)
    d = D
    pre = lambda x, h: f"{x} p3 dot {h} p4 dot add p5 add"  # noqa: E731
    # step 1 state programs (recomputed where needed; fan-out sums the grads)
    c1 = (f"{pre('p0', 'p1')} slice:1:{d}:{d} sigmoid p2 mul "
          f"{pre('p0', 'p1')} slice:1:0:{d} sigmoid {pre('p0', 'p1')} slice:1:{3 * d}:{d} tanh mul add")
    h1 = f"{c1} tanh {pre('p0', 'p1')} slice:1:{2 * d}:{d} sigmoid mul"
    # step 2: x2 is p6; its pre uses h1
    pre2 = f"p6 p3 dot {h1} p4 dot add p5 add"
    c2 = (f"{pre2} slice:1:{d}:{d} sigmoid {c1} mul {pre2} slice:1:0:{d} sigmoid "
          f"{pre2} slice:1:{3 * d}:{d} tanh mul add")
    h2 = f"{c2} tanh {pre2} slice:1:{2 * d}:{d} sigmoid mul"
    rng = np.random.default_rng(11)
    G = rng.uniform(-1, 1, (B, d)).astype(np.float32)
    ro, rg = R.op_program(h2, ins + [x2], G)
    M.set_precision("fp32")
    try:
        g = M.ExpressionGraph(1)
        ps = [g.param(f"p{i}", list(a.shape), np.ascontiguousarray(a))
              for i, a in enumerate(ins + [x2])]
        s1 = g.lstm_cell(ps[0], ps[1], ps[2], ps[3], ps[4], ps[5])
        s2 = g.lstm_cell(ps[6], g.lstm_state(s1), g.lstm_cell_state(s1), ps[3], ps[4], ps[5])
        out = g.lstm_state(s2)
        loss = g.reduce(M.ReduceOp.Sum, g.reshape(g.mul(out, g.constant(G)), [1, B * d]), 1)
        g.forward()
        g.zero_grads()
        g.backward(loss)
        mo = out.val().reshape(B, d)
        mg = [g.param_grad(f"p{i}").reshape(a.shape) for i, a in enumerate(ins + [x2])]
    finally:
        M.set_precision("tf32")
    assert np.abs(mo - ro).max() <= 2e-6 * np.abs(ro).max()
    for a, b in zip(mg, rg):
        assert np.abs(a - b).max() <= 5e-6 * np.abs(b).max(), np.abs(a - b).max()
