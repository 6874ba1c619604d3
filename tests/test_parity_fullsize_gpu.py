"""Oracle parity at the BASELINE.json model dimensions, in both precisions.

For Transformer-base (6+6, d512, h8, V32k), Transformer-big (d1024, h16,
ff4096), the Nematus shallow GRU (e512, d1024, V50k) and the deep-transition
GRU with layer norm (same dims): one synthetic batch small enough for the
unmodified reference (oracle/_ref) to finish its CPU step in under a minute,
same seeded parameters (bit-exact), then

* loss:      rel <= 1e-5 (FP32) / 2e-3 (TF32);
* gradients: per tensor ||d|| <= 1e-4 ||g_ref|| (FP32) / 1e-2 ||g_ref|| (TF32),
             absolute floor only for exactly-zero gradients (tests/parity_util.py);
* one Adam+EMA step (train.cpp:30-79): FP32 |d| <= 1e-3 lr on >= 99.9 % of
  elements; TF32 step-sign agreement >= 99 % where |g| is not negligible.

Reference: src/models.cpp:140-500 (model wiring), src/graph.cpp:648-924
(GRU, CE), src/train.cpp:30-79 (Adam, EMA).
"""
import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import CONFIGS, config_text, mtk as M, synth
from parity_util import check_adam_fp32, check_adam_sign, check_grads

pytestmark = pytest.mark.gpu

CASES = {"base": 4, "big": 2, "shallow": 2, "deep": 2}
LR = 3e-4 * 1 / 16000  # lr(step 1) of the default schedule (train.cpp:61-67)
LOSS_TOL = {"fp32": 1e-5, "tf32": 2e-3}

_ref_cache = {}


def ref_state(name):
    if name in _ref_cache:
        return _ref_cache[name]
    _ref_cache.clear()  # one model's state at a time (big: ~4 GB of host arrays)
    spec = CONFIGS[name]
    cfg = config_text(**spec)
    n = CASES[name]
    src, tgt = synth.corpus(n, spec["vocab"])
    ref = R.RefModel(cfg, 1)
    bs = R.BatchSet(R.Examples(src, tgt), n * 66, 1)
    assert bs.count == 1
    names = ref.param_names()
    init = {k: ref.param(k) for k in names}
    loss, tokens = ref.loss_grads(bs, 0, 1)
    grads = {k: ref.grad(k) for k in names}
    ref.adam_update(LR)
    after = {k: ref.param(k) for k in names}
    avg = {k: ref.state("avg", k) for k in names}
    st = dict(cfg=cfg, src=src, tgt=tgt, n=n, names=names, init=init, loss=loss, tokens=tokens,
              grads=grads, after=after, avg=avg)
    _ref_cache[name] = st
    return st


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
@pytest.mark.parametrize("name", list(CASES))
def test_step_parity_at_baseline_dims(cuda, name, prec):
    st = ref_state(name)
    M.set_precision(prec)
    try:
        ex = M.Examples([list(map(int, s)) for s in st["src"]], [list(map(int, t)) for t in st["tgt"]])
        batch = M.make_batches(ex, st["n"] * 66, 1, True)[0]
        assert batch.target_tokens() == st["tokens"]
        model = M.Model(st["cfg"])
        g = M.ExpressionGraph(1)
        model.register_params(g)
        names = st["names"]
        assert list(g.param_names()) == names
        for k in names:  # seeded init is bit-exact (graph.cpp:35-45, 100-122)
            assert np.array_equal(g.param_value(k), st["init"][k]), k
        g.clear()
        g.set_seed(1)
        loss = model.build_loss(g, batch)
        g.forward()
        g.zero_grads()
        g.backward(loss)
        value = float(loss.val()[0])
        rel = abs(value - st["loss"]) / abs(st["loss"])
        print(f"[parity] {name} {prec}: loss {value:.7f} ref {st['loss']:.7f} rel {rel:.2e}")
        assert rel <= LOSS_TOL[prec], (value, st["loss"])
        mine = {k: g.param_grad(k) for k in names}
        check_grads(names, mine, st["grads"], prec, name)
        adam = M.Adam(M.adam_defaults_for(st["cfg"]))
        avg = M.AveragedParameters(0.9999)
        adam.update(g, LR, avg)
        after = {k: g.param_value(k) for k in names}
        if prec == "fp32":
            check_adam_fp32(names, after, st["after"], LR)
            for k in names:
                assert np.allclose(avg.value(g, k), st["avg"][k], rtol=0, atol=1e-6), k
        else:
            check_adam_sign(names, st["init"], after, st["after"], st["grads"])
    finally:
        M.set_precision("tf32")
