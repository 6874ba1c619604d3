"""Quick end-to-end check: tiny Transformer, one batch, loss/grads vs reference."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import refbind as R
from paper_1804_00344_b200 import CONFIGS, config_text, mtk as M, synth

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
M.set_precision(prec)
cfg = config_text(**CONFIGS["tiny"])
src, tgt = synth.corpus(64, 8000)
ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
batches = M.make_batches(ex, 64 * 66, 1, True)
print("batches", len(batches), batches[0].rows(), batches[0].target_tokens())

ref = R.RefModel(cfg, 1)
rbs = R.BatchSet(R.Examples(src, tgt), 64 * 66, 1)
t = time.time()
rl, rt = ref.loss_grads(rbs, 0, 1)
print("ref loss", rl, "tokens", rt, "cpu s", time.time() - t)

model = M.Model(cfg)
g = M.ExpressionGraph(1)
model.register_params(g)
g.clear()
names = g.param_names()
assert names == ref.param_names(), "param order differs"
maxinit = max(np.abs(g.param_value(n) - ref.param(n)).max() for n in names)
print("init max diff", maxinit)
g.set_seed(1)
loss = model.build_loss(g, batches[0])
g.forward()
g.zero_grads()
g.backward(loss)
l = float(loss.val()[0])
print("mine loss", l, "rel", abs(l - rl) / abs(rl))
worst = 0
for n in names:
    a, b = g.param_grad(n), ref.grad(n)
    rel = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
    worst = max(worst, rel)
    if rel > 1e-3:
        print("  grad", n, rel)
print("worst grad rel-norm", worst)
M.sync()
t = time.time()
for _ in range(5):
    g.clear()
    loss = model.build_loss(g, batches[0])
    g.forward()
    g.zero_grads()
    g.backward(loss)
M.sync()
print("fwd+bwd ms", (time.time() - t) / 5 * 1e3)
