"""Full training-step parity on the B200 against the unmodified reference.

Config 1 of BASELINE.json (tiny Transformer 2+2, d256, h4, V8k, tied,
dropout 0) on the synthetic 64-sentence batch (B=64, S=T=33, 1,619 target
tokens): same batching, same seeded initial parameters (bit-exact), then
loss, every parameter gradient and the parameters after one Adam+EMA update
are compared with oracle/_ref.

Stated tolerances (tests/parity_util.py):
  loss rel <= 1e-5 (FP32 GEMMs, reference arithmetic) / 2e-3 (TF32 tensor
  cores); per-tensor gradient ||d||_2 <= 1e-4 ||g_ref||_2 (FP32) / 1e-2
  ||g_ref||_2 (TF32), with an absolute floor only for exactly-zero gradients
  (attention key biases); parameters after Adam: FP32 |d| <= 1e-3 * lr for
  >= 99.9 % of elements and <= 2 lr everywhere (step 1 moves every element by
  ~lr*sign(g), so elements whose |g| is near eps = 1e-9 flip with tiny
  gradient noise); TF32 step-sign agreement >= 99 % where |g| is not
  negligible.
"""
import numpy as np
import pytest

from oracle import refbind as R
from oracle import restate as S
from paper_1804_00344_b200 import CONFIGS, config_text, mtk as M, synth
from parity_util import check_adam_fp32, check_adam_sign, check_grads

pytestmark = pytest.mark.gpu

CFG = config_text(**CONFIGS["tiny"])


@pytest.fixture(scope="module")
def ref_state():
    src, tgt = synth.corpus(64, 8000)
    ref = R.RefModel(CFG, 1)
    bs = R.BatchSet(R.Examples(src, tgt), 64 * 66, 1)
    assert bs.count == 1
    loss, tokens = ref.loss_grads(bs, 0, 1)
    names = ref.param_names()
    grads = {n: ref.grad(n) for n in names}
    init = {n: ref.param(n) for n in names}
    lr = 3e-4 * 1 / 16000
    ref.adam_update(lr)
    after = {n: ref.param(n) for n in names}
    avg = {n: ref.state("avg", n) for n in names}
    return dict(src=src, tgt=tgt, loss=loss, tokens=tokens, names=names, grads=grads, init=init,
                after=after, avg=avg, lr=lr)


def _mine(prec, ref_state):
    M.set_precision(prec)
    src, tgt = ref_state["src"], ref_state["tgt"]
    ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
    batch = M.make_batches(ex, 64 * 66, 1, True)[0]
    model = M.Model(CFG)
    g = M.ExpressionGraph(1)
    model.register_params(g)
    g.clear()
    g.set_seed(1)
    loss = model.build_loss(g, batch)
    g.forward()
    g.zero_grads()
    g.backward(loss)
    return model, g, batch, float(loss.val()[0])


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_tiny_transformer_step_parity(cuda, ref_state, prec):
    model, g, batch, loss = _mine(prec, ref_state)
    names = ref_state["names"]
    assert list(g.param_names()) == names  # creation order == Adam/MTK1 order
    assert batch.target_tokens() == ref_state["tokens"] == 1619
    rel_loss = abs(loss - ref_state["loss"]) / abs(ref_state["loss"])
    assert rel_loss <= (1e-5 if prec == "fp32" else 2e-3), rel_loss
    check_grads(names, {n: g.param_grad(n) for n in names}, ref_state["grads"], prec, "tiny")
    # one Adam + EMA update (train.cpp:270-272) on the same gradients
    adam = M.Adam(M.adam_defaults_for(CFG))
    avg = M.AveragedParameters(0.9999)
    adam.update(g, ref_state["lr"], avg)
    after = {n: g.param_value(n) for n in names}
    if prec == "fp32":
        check_adam_fp32(names, after, ref_state["after"], ref_state["lr"])
        for n in names:
            assert np.allclose(avg.value(g, n), ref_state["avg"][n], rtol=0, atol=1e-6), n
    else:
        check_adam_sign(names, ref_state["init"], after, ref_state["after"], ref_state["grads"])


def test_init_bitexact(cuda, ref_state):
    M.set_precision("fp32")
    model = M.Model(CFG)
    g = M.ExpressionGraph(1)
    model.register_params(g)
    for n in ref_state["names"]:
        assert np.array_equal(g.param_value(n), ref_state["init"][n]), n


def test_step_is_bitwise_deterministic(cuda):
    """Two runs of the same update are bitwise identical (acceptance
    criterion 10; no unordered atomics on the default path)."""
    M.set_precision("tf32")
    cfg = config_text(arch="transformer", vocab=500, emb=128, heads=4, layers=2)
    ex = M.synth_examples(200, 500)
    batches = M.make_batches(ex, 2000, 1, True)

    def run():
        model = M.Model(cfg)
        g = M.ExpressionGraph(1)
        model.register_params(g)
        g.clear()
        adam = M.Adam(M.adam_defaults_for(cfg))
        avg = M.AveragedParameters()
        opts = M.TrainOptions()
        st = M.SyncStepper(model, g, adam, avg, opts)
        losses = [st.update([batches[i]], i, True).loss for i in range(3)]
        return losses, {n: g.param_value(n) for n in g.param_names()}

    l1, p1 = run()
    l2, p2 = run()
    assert l1 == l2
    for n in p1:
        assert np.array_equal(p1[n], p2[n]), n


def test_two_workers_equal_reference_train(cuda):
    """Synchronous 2-worker update (one GPU runs both workers in order) vs the
    reference's threaded trainSync: same batches, token-weighted combine,
    Adam + EMA (train.cpp:200-300); FP32 mode, <= 1e-6 relative like the
    reference's own DP test (test_train.cpp:237-242)."""
    M.set_precision("fp32")
    cfg = config_text(arch="transformer", vocab=60, emb=32, heads=2, layers=1)
    src, tgt = synth.corpus(40, 60)
    ref = R.RefModel(cfg, 9)
    ref.train(R.Examples(src, tgt), workers=2, budget=5 * 66, seed=9, epochs=1, max_updates=2)
    model = M.Model(cfg)
    g = M.ExpressionGraph(9)
    adam = M.Adam(M.adam_defaults_for(cfg))
    avg = M.AveragedParameters()
    opts = M.TrainOptions()
    opts.workers = 2
    opts.token_budget = 5 * 66
    opts.seed = 9
    opts.max_updates = 2
    res, _ = M.train(model, M.Examples([list(map(int, s)) for s in src],
                                       [list(map(int, t)) for t in tgt]), g, adam, avg, opts)
    assert res.updates == 2
    for n in ref.param_names():
        a, b = g.param_value(n), ref.param(n)
        assert np.allclose(a, b, rtol=1e-6, atol=1e-6 * max(1.0, np.abs(b).max())), n
    M.set_precision("tf32")


def test_dp_weights_match_restatement():
    """Worker seeds and weights used by the stepper follow train.cpp."""
    assert M.mix_seed(9, 1, 1) == S.mix_seed(9, 1, 1)


@pytest.mark.parametrize("arch,ln", [("s2s-shallow", False), ("s2s-deep", True), ("s2s-deep", False)])
def test_rnn_step_parity(cuda, arch, ln):
    """Nematus-style shallow and deep-transition RNNs (models.cpp:140-391):
    bidirectional GRU encoder, conditional GRU decoder with Bahdanau
    attention, readout, tied output layer; loss and all gradients vs the
    reference on one synthetic batch (FP32 GEMMs)."""
    M.set_precision("fp32")
    cfg = config_text(arch=arch, vocab=60, emb=16, state=24, layer_norm=ln)
    src, tgt = synth.corpus(6, 60)
    ref = R.RefModel(cfg, 3)
    bs = R.BatchSet(R.Examples(src, tgt), 6 * 66, 1)
    rl, _ = ref.loss_grads(bs, 0, 1)
    model = M.Model(cfg)
    g = M.ExpressionGraph(3)
    model.register_params(g)
    g.clear()
    assert list(g.param_names()) == ref.param_names()
    batch = M.make_batches(M.Examples([list(map(int, s)) for s in src],
                                      [list(map(int, t)) for t in tgt]), 6 * 66, 1, True)[0]
    loss = model.build_loss(g, batch)
    g.forward()
    g.zero_grads()
    g.backward(loss)
    l = float(loss.val()[0])
    assert abs(l - rl) <= 1e-5 * abs(rl), (l, rl)
    names = ref.param_names()
    check_grads(names, {n: g.param_grad(n) for n in names}, {n: ref.grad(n) for n in names},
                "fp32", f"{arch}{'-ln' if ln else ''}-toy")
    M.set_precision("tf32")


def test_pipelined_updates_equal_synchronous(cuda):
    """SyncStepper.update_pipelined returns each update's loss one call late;
    losses and parameters equal the synchronous update() sequence bitwise."""
    cfg = config_text(arch="transformer", vocab=200, emb=64, heads=4, layers=1)
    src, tgt = synth.corpus(48, 200)
    ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
    batches = M.make_batches(ex, 8 * 66, 1, True)

    def run(pipelined):
        model = M.Model(cfg)
        g = M.ExpressionGraph(3)
        model.register_params(g)
        g.clear()
        adam = M.Adam(M.adam_defaults_for(cfg))
        avg = M.AveragedParameters()
        opts = M.TrainOptions()
        opts.token_budget = 8 * 66
        st = M.SyncStepper(model, g, adam, avg, opts)
        losses = []
        for u in range(4):
            if pipelined:
                r = st.update_pipelined([batches[u]], u)
                if u > 0:
                    losses.append(r.loss)
            else:
                losses.append(st.update([batches[u]], u, True).loss)
        if pipelined:
            losses.append(st.flush_pipelined().loss)
        return losses, {n: g.param_value(n).copy() for n in g.param_names()}

    l1, p1 = run(False)
    l2, p2 = run(True)
    assert l1 == l2
    for n in p1:
        assert np.array_equal(p1[n], p2[n]), n


def test_async_one_worker_equals_reference_train_async(cuda):
    """trainAsync (train.cpp:302-404) with one worker is deterministic: the
    B200 rounds schedule must reproduce the reference's parameters after
    three updates (FP32 mode, the DP tolerance of test_train.cpp:237-242)."""
    M.set_precision("fp32")
    cfg = config_text(arch="transformer", vocab=60, emb=32, heads=2, layers=1)
    src, tgt = synth.corpus(40, 60)
    ref = R.RefModel(cfg, 9)
    ref.train(R.Examples(src, tgt), workers=1, budget=5 * 66, seed=9, epochs=1, max_updates=3,
              async_=True)
    model = M.Model(cfg)
    g = M.ExpressionGraph(9)
    adam = M.Adam(M.adam_defaults_for(cfg))
    avg = M.AveragedParameters()
    opts = M.TrainOptions()
    opts.workers = 1
    opts.async_ = True
    opts.token_budget = 5 * 66
    opts.seed = 9
    opts.max_updates = 3
    res, _ = M.train(model, M.Examples([list(map(int, s)) for s in src],
                                       [list(map(int, t)) for t in tgt]), g, adam, avg, opts)
    assert res.updates == 3
    for n in ref.param_names():
        a, b = g.param_value(n), ref.param(n)
        assert np.allclose(a, b, rtol=1e-6, atol=1e-6 * max(1.0, np.abs(b).max())), n
    M.set_precision("tf32")


def test_async_workers_stale_reads(cuda):
    """Several asynchronous workers (rounds of W stale reads, updates in
    worker order): every batch is consumed once, the step count and the
    loss trajectory are sane, and the run is reproducible."""
    M.set_precision("tf32")
    cfg = config_text(arch="transformer", vocab=60, emb=32, heads=2, layers=1)
    src, tgt = synth.corpus(60, 60)
    ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])

    def run(workers):
        model = M.Model(cfg)
        g = M.ExpressionGraph(3)
        adam = M.Adam(M.adam_defaults_for(cfg))
        avg = M.AveragedParameters()
        opts = M.TrainOptions()
        opts.workers = workers
        opts.async_ = True
        opts.token_budget = 5 * 66
        opts.seed = 3
        res, _ = M.train(model, ex, g, adam, avg, opts)
        return res, np.concatenate([g.param_value(n).ravel() for n in g.param_names()])

    nb = len(M.make_batches(ex, 5 * 66, 3, True))
    r3, p3 = run(3)
    r3b, p3b = run(3)
    r1, p1 = run(1)
    assert r3.updates == r1.updates == nb
    assert np.isfinite(r3.final_loss)
    assert np.array_equal(p3, p3b)
    assert not np.array_equal(p3, p1)  # stale reads change the trajectory
