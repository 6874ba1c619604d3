"""Arena high-water mark under reset-and-replay (test_tensor.cpp:193-206) and
the embedding tying modes other than `all` (TyingMode none / source-target,
layers.cpp:27-55): parameter names, creation order, seeded init and a full
training step's loss and gradients against the reference."""
import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import config_text, mtk as M, synth
from parity_util import check_grads

pytestmark = pytest.mark.gpu


def test_arena_high_water_stable_under_replay(cuda):
    a = M.Arena(1 << 20)

    def replay():
        a.alloc(100)
        a.alloc(200)
        a.alloc(100)
        a.reset()

    replay()
    hw = a.high_water_bytes()
    for _ in range(10):
        replay()
    assert a.high_water_bytes() == hw
    assert a.outstanding_bytes() == 0


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
@pytest.mark.parametrize("arch,tying", [("transformer", "none"), ("transformer", "source-target"),
                                        ("s2s-shallow", "none"), ("s2s-shallow", "source-target")])
def test_tying_modes_step_parity(cuda, arch, tying, prec):
    spec = dict(arch=arch, vocab=400, emb=64, state=96, heads=2, layers=2, tying=tying)
    cfg = config_text(**spec)
    n = 10
    src, tgt = synth.corpus(n, 400)
    ref = R.RefModel(cfg, 1)
    bs = R.BatchSet(R.Examples(src, tgt), n * 66, 1)
    names = ref.param_names()
    init = {k: ref.param(k) for k in names}
    rloss, rtok = ref.loss_grads(bs, 0, 1)
    M.set_precision(prec)
    try:
        ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
        batch = M.make_batches(ex, n * 66, 1, True)[0]
        model = M.Model(cfg)
        g = M.ExpressionGraph(1)
        model.register_params(g)
        assert list(g.param_names()) == names
        assert any(k.startswith("emb.E") and k != "emb.E" for k in names)  # untied tables exist
        for k in names:
            assert np.array_equal(g.param_value(k), init[k]), k
        g.clear()
        g.set_seed(1)
        loss = model.build_loss(g, batch)
        g.forward()
        g.zero_grads()
        g.backward(loss)
        value = float(loss.val()[0])
        assert abs(value - rloss) <= (1e-5 if prec == "fp32" else 2e-3) * abs(rloss)
        check_grads(names, {k: g.param_grad(k) for k in names},
                    {k: ref.grad(k) for k in names}, prec, f"tying-{arch}-{tying}")
    finally:
        M.set_precision("tf32")
