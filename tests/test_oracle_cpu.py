"""Pins the oracle before it is trusted (CPU only).

1. The unmodified reference (oracle/_ref) reproduces the known-answer values
   of the reference's own test suites (tests/test_tensor.cpp,
   test_graph.cpp, test_train.cpp; file:line cited per case).
2. The numpy restatement (oracle/restate.py) agrees with oracle/_ref on
   random instances of every op it restates.
"""
import math

import numpy as np
import pytest

from oracle import refbind as R
from oracle import restate as S

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


# ------------------------------------------------ reference known answers

def test_kat_matmul():  # test_tensor.cpp:19-31
    a = np.array([[1, 2], [3, 4]], np.float32)
    b = np.array([[5, 6], [7, 8]], np.float32)
    assert R.matmul(a, b).tolist() == [[19, 22], [43, 50]]
    assert R.matmul(np.eye(2, dtype=np.float32), a).tolist() == a.tolist()


def test_kat_softmax():  # test_tensor.cpp:141-171
    out, _ = R.op_softmax(np.array([[1, 2, 3]], np.float32), None, np.zeros((1, 3), np.float32))
    assert np.allclose(out[0], [0.09003, 0.24473, 0.66524], atol=1e-5)
    out, _ = R.op_softmax(np.array([[1000, 1000]], np.float32), None, np.zeros((1, 2), np.float32))
    assert np.allclose(out, 0.5)
    with pytest.raises(R.RefError) as e:
        R.op_softmax(np.array([[1, 2, 3], [4, 5, 6]], np.float32),
                     np.array([[0, 0, 0], [1, 1, 1]], np.float32), np.zeros((2, 3), np.float32))
    assert e.value.kind == "NumericError"


def test_kat_layernorm():  # test_graph.cpp:170-191
    x = np.array([[1, 2, 3]], np.float32)
    out, *_ = R.op_layernorm(x, np.ones(3), np.zeros(3), np.zeros((1, 3)))
    assert np.allclose(out, [[-1.22474, 0, 1.22474]], atol=1e-5)
    out, *_ = R.op_layernorm(np.full((1, 4), 7, np.float32), np.ones(4), np.full(4, 0.5),
                             np.zeros((1, 4)))
    assert np.allclose(out, 0.5)


def test_kat_cross_entropy():  # test_graph.cpp:226-249
    loss, _ = R.op_xent(np.zeros((1, 1, 4), np.float32), np.array([[2]]), None)
    assert abs(loss - math.log(4)) < 1e-6
    lg = np.zeros((1, 1, 4), np.float32)
    lg[0, 0, 1] = 1000
    loss, _ = R.op_xent(lg, np.array([[1]]), None)
    assert abs(loss) < 1e-6
    with pytest.raises(R.RefError) as e:
        R.op_xent(np.zeros((1, 1, 4), np.float32), np.array([[7]]), None)
    assert e.value.kind == "DataError"


def test_kat_gru_zero_weights():  # test_graph.cpp:136-168
    e = d = 2
    w = np.zeros(3 * d * d + 3 * d + 3 * e * d, np.float32)
    out, *_ = R.op_gru(np.zeros((1, 2)), np.ones((1, 2)), w, False, np.zeros((1, 2)), e, d)
    assert np.allclose(out, 0)
    out, *_ = R.op_gru(np.ones((1, 2)), np.zeros((1, 2)), w, False, np.zeros((1, 2)), e, d)
    assert np.allclose(out, 0.5)


def test_kat_parameter_census():  # SURVEY 8(a) a2 (reference parameterTotal)
    from paper_1804_00344_b200 import CONFIGS, config_text
    assert R.parameter_total(config_text(**CONFIGS["tiny"])) == 5_743_424


# ------------------------------------------- restatement vs the reference

def test_restate_layernorm():
    rng = np.random.default_rng(0)
    x = rng.normal(size=(7, 33)).astype(np.float32)
    g, b = rng.normal(size=33).astype(np.float32), rng.normal(size=33).astype(np.float32)
    G = rng.normal(size=(7, 33)).astype(np.float32)
    out, gx, gg, gb = R.op_layernorm(x, g, b, G)
    o2, rs, xh = S.layernorm_fwd(x, g, b)
    dx, dg, db = S.layernorm_bwd(G, g, rs, xh)
    assert np.allclose(out, o2, atol=2e-6)
    assert np.allclose(gx, dx, atol=1e-5) and np.allclose(gg, dg, atol=1e-5)
    assert np.allclose(gb, db, atol=1e-5)


def test_restate_softmax_masked():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(3, 4, 9)).astype(np.float32) * 5
    m = (rng.random((3, 1, 9)) > 0.3).astype(np.float32)
    m[..., 0] = 1
    G = rng.normal(size=x.shape).astype(np.float32)
    out, gx = R.op_softmax(x, m, G)
    y = S.softmax_fwd(x, m)
    assert np.allclose(out, y, atol=1e-6)
    assert np.allclose(gx, S.softmax_bwd(y, G), atol=1e-6)
    assert np.all(out[np.broadcast_to(m, x.shape) == 0] == 0)


def test_restate_xent():
    rng = np.random.default_rng(2)
    lg = rng.uniform(-2, 2, (2, 3, 11)).astype(np.float32)
    t = rng.integers(0, 11, (2, 3))
    m = np.array([[1, 1, 0], [1, 1, 1]], np.float32)
    loss, g = R.op_xent(lg, t, m)
    l2, g2 = S.xent(lg, t, m)
    assert abs(loss - l2) < 1e-5 and np.allclose(g, g2, atol=1e-6)


@pytest.mark.parametrize("causal", [False, True])
def test_restate_mha_core(causal):
    rng = np.random.default_rng(3)
    b, t, d, h = 2, 5, 8, 2
    q, k, v = (rng.normal(size=(b, t, d)).astype(np.float32) for _ in range(3))
    km = np.ones((b, t), np.float32)
    km[1, 3:] = 0
    G = rng.normal(size=(b, t, d)).astype(np.float32)
    out, gq, gk, gv = R.op_mha(q, k, v, km, causal, h, G)
    o2, p = S.mha_core(q, k, v, km, causal, h)
    dq, dk, dv = S.mha_core_bwd(q, k, v, p, G, h)
    assert np.allclose(out, o2, atol=1e-5)
    assert np.allclose(gq, dq, atol=1e-5) and np.allclose(gk, dk, atol=1e-5)
    assert np.allclose(gv, dv, atol=1e-5)


@pytest.mark.parametrize("ln,e", [(False, 3), (True, 3), (True, 0)])
def test_restate_gru_forward(ln, e):
    rng = np.random.default_rng(4)
    b, d = 3, 5
    names = ["Uz", "Ur", "Uh", "bz", "br", "bh"] + (["Wz", "Wr", "Wx"] if e else [])
    if ln:
        names += ["lnGz", "lnBz", "lnGr", "lnBr"] + (["lnGx", "lnBx"] if e else [])
    shapes = {n: (d, d) if n[0] == "U" else (e, d) if n[0] == "W" else (d,) for n in names}
    W = {n: rng.normal(size=shapes[n]).astype(np.float32) * 0.5 for n in names}
    packed = np.concatenate([W[n].ravel() for n in names])
    h = rng.normal(size=(b, d)).astype(np.float32)
    x = rng.normal(size=(b, e)).astype(np.float32) if e else None
    out, *_ = R.op_gru(h, x, packed, ln, np.zeros((b, d)), e, d)
    assert np.allclose(out, S.gru_fwd(h, x, W, ln), atol=2e-6)


def test_restate_adam_kat():  # test_train.cpp:66-75 (theta 0 -> -0.1 -> -0.2)
    th, m, v = S.adam_step(np.zeros(1), np.ones(1), np.zeros(1), np.zeros(1), 0.1, 1)
    assert abs(th[0] + 0.1) < 1e-6
    th, m, v = S.adam_step(th, np.ones(1), m, v, 0.1, 2)
    assert abs(th[0] + 0.2) < 1e-6


def test_restate_lr_kat():  # test_train.cpp:115-125
    assert S.lr_schedule(0) == 0
    assert abs(S.lr_schedule(16000) - 3e-4) < 1e-9
    assert abs(S.lr_schedule(64000) - 1.5e-4) < 1e-9
    assert abs(S.lr_schedule(8000) - 1.5e-4) < 1e-9


def test_restate_dp_combine_matches_reference_two_workers():
    """Reference train() with 2 workers == restated combine of two
    single-batch gradients + one reference Adam step (train.cpp:254-272)."""
    from paper_1804_00344_b200 import config_text, synth
    cfg = config_text(arch="transformer", vocab=40, emb=16, heads=2, layers=1)
    src, tgt = synth.corpus(12, 40)
    ex = R.Examples(src, tgt)
    budget = 3 * 66
    a = R.RefModel(cfg, 1)
    a.train(ex, workers=2, budget=budget, seed=1, epochs=1, max_updates=1)
    bs = R.BatchSet(ex, budget, 1)
    w = R.RefModel(cfg, 1)
    grads, toks = [], []
    for i in range(2):
        _, t = w.loss_grads(bs, i, S.mix_seed(1, 0, i))
        grads.append({n: w.grad(n) for n in w.param_names()})
        toks.append(t)
    for n in w.param_names():
        w.set_grad(n, S.dp_combine([gr[n] for gr in grads], toks))
    w.adam_update(float(S.lr_schedule(1)))
    for n in w.param_names():
        assert np.array_equal(a.param(n), w.param(n)), n
