"""One attention forward+backward at Transformer-base shape (for ncu / timing)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1804_00344_b200 import mtk as M
b, t, d, h = int(os.environ.get("B", 250)), int(os.environ.get("T", 33)), 512, 8
rng = np.random.default_rng(0)
g = M.ExpressionGraph(1)
q = g.param("q", [b, t, d], rng.normal(size=(b, t, d)).astype(np.float32))
k = g.param("k", [b, t, d], rng.normal(size=(b, t, d)).astype(np.float32))
v = g.param("v", [b, t, d], rng.normal(size=(b, t, d)).astype(np.float32))
mask = np.ones((b, t), np.float32); mask[:, 25:] = 0
def run():
    g.clear()
    qq, kk, vv = g.param("q", [b, t, d]), g.param("k", [b, t, d]), g.param("v", [b, t, d])
    o = g.attention(qq, kk, vv, mask, True, h)
    loss = g.reduce(M.ReduceOp.Sum, g.reshape(o, [1, b * t * d]), 1)
    g.forward(); g.zero_grads(); g.backward(loss)
for _ in range(3): run()
M.sync()
M.prof_enable(True)
for _ in range(5): run()
print(M.prof_report())
