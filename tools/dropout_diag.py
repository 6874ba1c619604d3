"""Diagnose FP32 parity with / without host dropout masks (tiny-ish transformer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from oracle import refbind as R
from paper_1804_00344_b200 import config_text, mtk as M, synth
from parity_util import grad_ratios

M.set_dropout_rng("host")
M.set_precision("fp32")
for p in [0.1]:
    for spec in [dict(arch="transformer", vocab=8000, emb=256, heads=4, layers=2, dropout=p)]:
        cfg = config_text(**spec)
        n = 12
        src, tgt = synth.corpus(n, spec["vocab"])
        ref = R.RefModel(cfg, 1)
        bs = R.BatchSet(R.Examples(src, tgt), n * 66, 1)
        rloss, rtok = ref.loss_grads(bs, 0, 0x5EED)
        names = ref.param_names()
        rg = {k: ref.grad(k) for k in names}
        ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
        batch = M.make_batches(ex, n * 66, 1, True)[0]
        model = M.Model(cfg); g = M.ExpressionGraph(1); model.register_params(g); g.clear(); g.set_seed(0x5EED)
        loss = model.build_loss(g, batch); g.forward(); g.zero_grads(); g.backward(loss)
        rows, G = grad_ratios(names, {k: g.param_grad(k) for k in names}, rg)
        a = g.param_grad("dec.l1.ffn.b1"); b = rg["dec.l1.ffn.b1"]
        e = np.abs(a - b); idx = np.argsort(-e)[:8]
        print("b1 err top", [(int(i), float(e[i]), float(b[i])) for i in idx], "norm", float(np.linalg.norm(b)))
        A = g.param_grad("dec.l1.ffn.W1"); B = rg["dec.l1.ffn.W1"]
        ce = np.linalg.norm(A - B, axis=0); print("W1 cols with err>1e-6*norm:", int((ce > 1e-6 * np.linalg.norm(B)).sum()), "of", ce.size)
        print(f"p={p} emb={spec['emb']} loss {float(loss.val()[0]):.8f} ref {rloss:.8f}")
        if p > 0 and spec["emb"] == 256:
            for r in rows:
                if "dec.l1.ffn" in r[0]:
                    print("   ", r[0], f"{r[3]:.2e}")
        print("    median", np.median([r[3] for r in rows]))
