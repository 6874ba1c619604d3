"""Packed-row Transformer training step (TF32 mode; Model::buildLoss with
RowPacking + attentionPacked): every position-wise op runs over the real
tokens only.  Padding rows carry exactly zero gradient in the reference
(masked keys, masked loss rows), so the packed step must equal the padded
step up to TF32 rounding: loss and every parameter gradient against
MTK_PACK=0 (padded layout) and against the reference oracle.
"""
import os

import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import config_text, mtk as M, synth
from parity_util import check_grads

pytestmark = pytest.mark.gpu


def step(cfg, src, tgt, n, pack):
    os.environ["MTK_PACK"] = "1" if pack else "0"
    try:
        M.set_precision("tf32")
        ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
        batch = M.make_batches(ex, n * 66, 1, True)[0]
        model = M.Model(cfg)
        g = M.ExpressionGraph(1)
        model.register_params(g)
        g.clear()
        g.set_seed(1)
        loss = model.build_loss(g, batch)
        g.forward()
        g.zero_grads()
        g.backward(loss)
        names = g.param_names()
        return float(loss.val()[0]), {k: g.param_grad(k) for k in names}, names, g.node_count()
    finally:
        os.environ.pop("MTK_PACK", None)


@pytest.mark.parametrize("spec", [
    dict(arch="transformer", vocab=600, emb=128, heads=2, layers=2),
    dict(arch="transformer", vocab=600, emb=128, heads=2, layers=2, post_norm=True),
    dict(arch="transformer", vocab=8000, emb=256, heads=4, layers=2),
], ids=["prenorm", "postnorm", "tiny"])
def test_packed_equals_padded_and_reference(cuda, spec):
    n = 24
    cfg = config_text(**spec)
    src, tgt = synth.corpus(n, spec["vocab"])
    lp, gp, names, nodes_p = step(cfg, src, tgt, n, True)
    lu, gu, _, nodes_u = step(cfg, src, tgt, n, False)
    print(f"[pack] loss packed {lp:.7f} padded {lu:.7f}; nodes {nodes_p} vs {nodes_u}")
    assert nodes_p != nodes_u  # the packed path really ran
    assert abs(lp - lu) <= 2e-4 * abs(lu)
    check_grads(names, gp, gu, "tf32", "packed-vs-padded")
    ref = R.RefModel(cfg, 1)
    bs = R.BatchSet(R.Examples(src, tgt), n * 66, 1)
    rl, _ = ref.loss_grads(bs, 0, 1)
    assert abs(lp - rl) <= 2e-3 * abs(rl)
    check_grads(names, gp, {k: ref.grad(k) for k in names}, "tf32", "packed-vs-ref")
