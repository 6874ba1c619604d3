"""Persistent GRU scan (kernels/rnn_persist.cu) against the per-step launch
path (MTK_RNN_PERSIST=0: one grouped tcgen05 GEMM + gru/bahdanau kernels per
block and step) and against the reference oracle.

Both paths run the reference's arithmetic (gruCell graph.cpp:633-745,
Bahdanau layers.cpp:59-79) in TF32 mode; they differ only in the K order of
the recurrent products (K-split partials summed in a fixed order vs the GEMM
kernel's split-K), so loss and gradients agree to TF32 rounding.  Covered:
shallow (1+2 blocks, attention), deep transition with layer norm (4+8
blocks), b > 128 rows (two m-tiles), padding blend, both encoder directions
in one launch, determinism of the persistent path.
"""
import os

import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import config_text, mtk as M, synth
from parity_util import check_grads

pytestmark = pytest.mark.gpu

CASES = {
    "shallow-d256": (dict(arch="s2s-shallow", vocab=500, emb=128, state=256), 40),
    "deep-ln-d256": (dict(arch="s2s-deep", vocab=500, emb=128, state=256, layer_norm=True), 24),
    "shallow-b160": (dict(arch="s2s-shallow", vocab=300, emb=64, state=128), 160),
}


def step(spec, n, persist):
    os.environ["MTK_RNN_PERSIST"] = "1" if persist else "0"
    try:
        M.set_precision("tf32")
        cfg = config_text(**spec)
        src, tgt = synth.corpus(n, spec["vocab"])
        ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
        batch = M.make_batches(ex, n * 66, 1, True)[0]
        model = M.Model(cfg)
        g = M.ExpressionGraph(1)
        model.register_params(g)
        g.clear()
        g.set_seed(1)
        l0 = M.launch_count()
        loss = model.build_loss(g, batch)
        g.forward()
        g.zero_grads()
        g.backward(loss)
        value = float(loss.val()[0])
        launches = M.launch_count() - l0
        names = g.param_names()
        return value, {k: g.param_grad(k) for k in names}, names, launches, batch.rows()
    finally:
        os.environ.pop("MTK_RNN_PERSIST", None)


@pytest.mark.parametrize("name", list(CASES))
def test_persistent_scan_matches_per_step_path(cuda, name):
    spec, n = CASES[name]
    lp, gp, names, kp, rows = step(spec, n, True)
    ls, gs, _, ks, _ = step(spec, n, False)
    assert rows == n
    print(f"[persist] {name}: loss {lp:.7f} vs {ls:.7f}, launches {kp} vs {ks}")
    assert abs(lp - ls) <= 2e-4 * abs(ls)
    check_grads(names, gp, gs, "tf32", f"persist-{name}")
    assert kp < ks  # the recurrence is one launch per scan, not per step
    lp2, gp2, _, _, _ = step(spec, n, True)
    assert lp2 == lp and all(np.array_equal(gp[k], gp2[k]) for k in names)


@pytest.mark.parametrize("name", ["shallow-d256", "deep-ln-d256"])
def test_persistent_scan_vs_reference(cuda, name):
    spec, n = CASES[name]
    n = 8
    cfg = config_text(**spec)
    src, tgt = synth.corpus(n, spec["vocab"])
    ref = R.RefModel(cfg, 1)
    bs = R.BatchSet(R.Examples(src, tgt), n * 66, 1)
    rloss, _ = ref.loss_grads(bs, 0, 1)
    names = ref.param_names()
    lp, gp, mine_names, _, _ = step(spec, n, True)
    assert list(mine_names) == names
    assert abs(lp - rloss) <= 2e-3 * abs(rloss), (lp, rloss)
    check_grads(names, gp, {k: ref.grad(k) for k in names}, "tf32", f"persist-ref-{name}")
