"""Remaining model zoo (row f4; reference models.cpp:504-623, 678-745):
`lm` (decoder only, no encoder), `hard-att` (monotone hard attention: the
gate is realised mid-graph and read on the host to move each row's source
pointer), `ape-dual` (two deep RNN encoders over two
source streams, one deep RNN decoder), and `custom` compositions (comma-
separated encoder kinds + a decoder kind: multi-source Transformer and
mixed Transformer/RNN encoders feeding an RNN decoder through the ctxW
combiner).  Same seeded parameters as the reference (bit-exact, in the
reference's creation order), then loss and every parameter gradient against
oracle/_ref in FP32 (tests/parity_util.py bounds) and TF32.
"""
import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import mtk as M, synth
from parity_util import check_grads

pytestmark = pytest.mark.gpu


def cfg_text(arch, vocab=300, emb=32, state=48, heads=2, layers=1, layer_norm=0, enc="",
             dec="", arity=1):
    s = (f"architecture: {arch}\nsource-vocab: {vocab}\ntarget-vocab: {vocab}\nemb-dim: {emb}\n"
         f"state-dim: {state}\nheads: {heads}\nlayers: {layers}\ndropout: 0\ntying: all\n"
         f"layer-norm: {layer_norm}\npost-norm: 0\nsource-arity: {arity}\n")
    if enc:
        s += f"encoder-kind: {enc}\n"
    if dec:
        s += f"decoder-kind: {dec}\n"
    return s


CASES = {
    "lm": (cfg_text("lm"), 1),
    "hard-att": (cfg_text("hard-att"), 1),
    "hard-att-ln": (cfg_text("hard-att", layer_norm=1), 1),
    "ape-dual": (cfg_text("ape-dual", layer_norm=1, arity=2), 2),
    "custom-tf2": (cfg_text("custom", emb=64, state=64, enc="transformer,transformer",
                            dec="transformer", arity=2), 2),
    "custom-mixed": (cfg_text("custom", emb=64, state=64, enc="transformer,rnn-shallow",
                              dec="rnn-shallow", arity=2), 2),
}


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
@pytest.mark.parametrize("name", list(CASES))
def test_zoo_step_parity(cuda, name, prec):
    cfg, streams = CASES[name]
    n = 10
    src, tgt = synth.corpus(n, 300)
    extra = [[s[::-1].copy() for s in src]] if streams > 1 else []  # second source stream
    ref = R.RefModel(cfg, 1)
    budget = n * 33 * (streams + 1)
    bs = R.BatchSet(R.Examples(src, tgt, extra), budget, 1)
    assert bs.count == 1
    names = ref.param_names()
    init = {k: ref.param(k) for k in names}
    rloss, rtok = ref.loss_grads(bs, 0, 1)
    rgrads = {k: ref.grad(k) for k in names}
    M.set_precision(prec)
    try:
        ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt],
                        [[list(map(int, x)) for x in st] for st in extra])
        batch = M.make_batches(ex, budget, 1, True)[0]
        assert batch.target_tokens() == rtok
        model = M.Model(cfg)
        g = M.ExpressionGraph(1)
        model.register_params(g)
        assert list(g.param_names()) == names
        for k in names:
            assert np.array_equal(g.param_value(k), init[k]), k
        g.clear()
        g.set_seed(1)
        loss = model.build_loss(g, batch)
        g.forward()
        g.zero_grads()
        g.backward(loss)
        value = float(loss.val()[0])
        tol = 1e-5 if prec == "fp32" else 2e-3
        assert abs(value - rloss) <= tol * abs(rloss), (value, rloss)
        check_grads(names, {k: g.param_grad(k) for k in names}, rgrads, prec, f"zoo-{name}")
    finally:
        M.set_precision("tf32")
