"""Dropout (row a19): ExpressionGraph::dropoutMask / dropout (graph.cpp:817-846)
seeded per (update, worker) (train.cpp:170-176).

* Host RNG mode (the reference's own mt19937_64 draws, uploaded as constants):
  a full training step with dropout 0.1 matches the unmodified reference in
  FP32 mode -- the masks are bit-identical, so the usual FP32 step tolerances
  hold (loss rel <= 1e-5, per-tensor gradients, tests/parity_util.py).  Covers
  the Transformer's variational embedding dropout and sublayer dropout
  (models.cpp:210, layers.cpp:135) and the RNN's state/context masks
  (models.cpp:153-162, 302-304).
* Device mode (throughput; kernels/dropout.cu, Philox masks recomputed in the
  backward): keep rate, mask values {0, 1/(1-p)}, forward/backward use the
  same mask, variational masks are constant along their axis, the fused
  residual r + dropout(f) equals the unfused composition bitwise, and a model
  step is reproducible for a fixed seed.
"""
import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import config_text, mtk as M, synth
from parity_util import check_grads

pytestmark = pytest.mark.gpu


@pytest.fixture
def host_rng():
    M.set_dropout_rng("host")
    yield
    M.set_dropout_rng("auto")
    M.set_precision("tf32")


@pytest.fixture
def device_rng():
    M.set_dropout_rng("device")
    yield
    M.set_dropout_rng("auto")
    M.set_precision("tf32")


CASES = {
    # (small dims: a ReLU pre-activation within rounding distance of zero flips
    # with ulp-level differences upstream -- CUDA vs glibc expf in softmax --
    # and moves one hidden unit's gradient; at emb 256 / 12 sentences one
    # such flip puts dec.l1.ffn.W1 at 4e-3, unrelated to the masks)
    "transformer": dict(arch="transformer", vocab=2000, emb=128, heads=4, layers=2, dropout=0.1),
    "transformer-postnorm": dict(arch="transformer", vocab=500, emb=64, heads=4, layers=2,
                                 dropout=0.1, post_norm=True),
    "s2s-shallow": dict(arch="s2s-shallow", vocab=300, emb=32, state=48, dropout=0.1),
    "s2s-deep": dict(arch="s2s-deep", vocab=300, emb=32, state=48, dropout=0.1, layer_norm=True),
}


@pytest.mark.parametrize("name", list(CASES))
def test_host_masks_step_parity_fp32(cuda, host_rng, name):
    spec = CASES[name]
    cfg = config_text(**spec)
    n = 12
    src, tgt = synth.corpus(n, spec["vocab"])
    ref = R.RefModel(cfg, 1)
    bs = R.BatchSet(R.Examples(src, tgt), n * 66, 1)
    seed = 0x5EED
    rloss, rtok = ref.loss_grads(bs, 0, seed)
    names = ref.param_names()
    rgrads = {k: ref.grad(k) for k in names}
    # the same batch without dropout gives clearly different gradients (masks are live)
    ref0 = R.RefModel(config_text(**dict(spec, dropout=0.0)), 1)
    ref0.loss_grads(bs, 0, seed)
    g0 = np.concatenate([ref0.grad(k).ravel() for k in names])
    g1 = np.concatenate([rgrads[k].ravel() for k in names])
    assert np.linalg.norm(g0 - g1) > 1e-2 * np.linalg.norm(g1)

    M.set_precision("fp32")
    ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
    batch = M.make_batches(ex, n * 66, 1, True)[0]
    assert batch.target_tokens() == rtok
    model = M.Model(cfg)
    g = M.ExpressionGraph(1)
    model.register_params(g)
    g.clear()
    g.set_seed(seed)
    loss = model.build_loss(g, batch)
    g.forward()
    g.zero_grads()
    g.backward(loss)
    value = float(loss.val()[0])
    assert abs(value - rloss) <= 1e-5 * abs(rloss), (value, rloss)
    check_grads(names, {k: g.param_grad(k) for k in names}, rgrads, "fp32", f"dropout-{name}")


def _graph_with(x):
    g = M.ExpressionGraph(1)
    g.set_seed(77)
    xp = g.param("x", list(x.shape), np.ascontiguousarray(x, np.float32))
    return g, xp


def _sum_all(g, y):
    r = y
    while len(r.shape) > 1:
        r = g.reduce(M.ReduceOp.Sum, r, len(r.shape) - 1)
    return g.reduce(M.ReduceOp.Sum, r, 0, True)


@pytest.mark.parametrize("axis", [-1, 1])
def test_device_dropout_forward_backward_same_mask(cuda, device_rng, axis):
    rng = np.random.default_rng(0)
    x = rng.uniform(0.5, 1.5, size=(16, 24, 64)).astype(np.float32)
    p = 0.1
    g, xp = _graph_with(x)
    y = g.dropout(xp, p, axis)
    loss = _sum_all(g, y)
    g.forward()
    g.zero_grads()
    g.backward(loss)
    yv = y.val().reshape(x.shape)
    m = g.param_grad("x").reshape(x.shape)  # d sum(x*m) / dx = m
    keep = np.float32(1) / (np.float32(1) - np.float32(p))
    assert set(np.unique(m).tolist()) <= {0.0, float(keep)}
    np.testing.assert_array_equal(yv, x * m)
    frac = float((m == 0).mean())
    sd = np.sqrt(p * (1 - p) / (m.size if axis < 0 else m.size / x.shape[1]))
    assert abs(frac - p) < 6 * sd, frac
    if axis == 1:  # one mask per (row, feature), broadcast along axis 1
        assert np.array_equal(m, np.broadcast_to(m[:, :1, :], m.shape))
    else:
        assert not np.array_equal(m[:, 0, :], m[:, 1, :])


def test_device_dropout_reproducible_and_seeded(cuda, device_rng):
    x = np.ones((64, 128), np.float32)

    def mask(seed):
        g = M.ExpressionGraph(1)
        g.set_seed(seed)
        m = g.dropout_mask([64, 128], 0.25)
        g.forward()
        return m.val().copy()

    a, b, c = mask(5), mask(5), mask(6)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)
    assert abs(float((a == 0).mean()) - 0.25) < 0.03
    del x


def test_device_dropout_residual_fused_equals_unfused(cuda, device_rng):
    rng = np.random.default_rng(1)
    r = rng.standard_normal((40, 96)).astype(np.float32)
    f = rng.standard_normal((40, 96)).astype(np.float32)
    w = rng.standard_normal((40, 96)).astype(np.float32)

    def run(fused):
        g = M.ExpressionGraph(1)
        g.set_seed(3)
        rp = g.param("r", [40, 96], r)
        fp = g.param("f", [40, 96], f)
        wc = g.constant(w)
        fx = g.tanh(fp)
        d = g.dropout(fx, 0.3)
        y = g.residual_add(rp, d) if fused else g.add(rp, d)
        loss = _sum_all(g, g.mul(y, wc))
        g.forward()
        g.zero_grads()
        g.backward(loss)
        return y.val().copy(), g.param_grad("r"), g.param_grad("f")

    a, b = run(True), run(False)
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)


@pytest.mark.parametrize("arch", ["transformer", "s2s-shallow"])
def test_device_dropout_model_step(cuda, device_rng, arch):
    M.set_precision("tf32")
    spec = dict(arch=arch, vocab=400, emb=64, state=96, heads=4, layers=2)
    ex = M.synth_examples(48, 400)
    batch = M.make_batches(ex, 48 * 66, 1, True)[0]

    def step(p, seed):
        cfg = config_text(**dict(spec, dropout=p))
        model = M.Model(cfg)
        g = M.ExpressionGraph(1)
        model.register_params(g)
        g.clear()
        g.set_seed(seed)
        loss = model.build_loss(g, batch)
        g.forward()
        g.zero_grads()
        g.backward(loss)
        names = g.param_names()
        return float(loss.val()[0]), np.concatenate([g.param_grad(k).ravel() for k in names])

    l1, g1 = step(0.1, 11)
    l2, g2 = step(0.1, 11)
    l3, _ = step(0.1, 12)
    l0, _ = step(0.0, 11)
    assert np.isfinite(l1) and l1 == l2 and np.array_equal(g1, g2)
    assert l1 != l3 and l1 != l0
