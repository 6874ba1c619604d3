"""Isolate the FP32 FFN + dropout gradient discrepancy: x -> LN -> affineRelu -> affine -> *mask -> +x -> LN -> sum(out*G),
vs float64 numpy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1804_00344_b200 import mtk as M

M.set_precision(sys.argv[1] if len(sys.argv) > 1 else "fp32")
M.set_dropout_rng("host")
rng = np.random.default_rng(0)
N, d = int(os.environ.get("N", 400)), int(os.environ.get("D", 256))
x = rng.standard_normal((N, d)).astype(np.float32)
W1 = (rng.standard_normal((d, 4 * d)) * 0.05).astype(np.float32)
b1 = (rng.standard_normal(4 * d) * 0.05).astype(np.float32)
W2 = (rng.standard_normal((4 * d, d)) * 0.05).astype(np.float32)
b2 = np.zeros(d, np.float32)
G = rng.standard_normal((N, d)).astype(np.float32)
keep = np.float32(1) / np.float32(0.9)
mask = np.where(rng.uniform(size=(N, d)) >= 0.1, keep, np.float32(0)).astype(np.float32)

def ln(v):
    mu = v.mean(-1, keepdims=True); var = ((v - mu) ** 2).mean(-1, keepdims=True)
    return (v - mu) / np.sqrt(var + 1e-9), 1 / np.sqrt(var + 1e-9)

def ref(use_mask, final_ln):
    X = x.astype(np.float64)
    xh, rs = ln(X)
    a = xh @ W1 + b1; h = np.maximum(a, 0)
    y = h @ W2 + b2
    m = mask if use_mask else 1.0
    z = X + y * m
    if final_ln:
        zh, rs2 = ln(z); out = zh
        # LN backward with g=1, b=0
        dzh = G.astype(np.float64)
        dz = rs2 * (dzh - dzh.mean(-1, keepdims=True) - zh * (dzh * zh).mean(-1, keepdims=True))
    else:
        dz = G.astype(np.float64)
    dy = dz * m
    dW2 = h.T @ dy
    dh = dy @ W2.T * (a > 0)
    dW1 = xh.T @ dh
    return dW1, dW2

for use_mask in [False, True]:
    for final_ln in [False, True]:
        g = M.ExpressionGraph(1)
        xp = g.param("x", [N, d], x)
        w1 = g.param("W1", [d, 4 * d], W1); bb1 = g.param("b1", [4 * d], b1)
        w2 = g.param("W2", [4 * d, d], W2); bb2 = g.param("b2", [d], b2)
        ones = g.param("g1", [d], np.ones(d, np.float32)); zeros = g.param("z1", [d], np.zeros(d, np.float32))
        ones2 = g.param("g2", [d], np.ones(d, np.float32)); zeros2 = g.param("z2", [d], np.zeros(d, np.float32))
        xn = g.layer_norm(xp, ones, zeros)
        y = g.affine(g.affine_relu(xn, w1, bb1) if os.environ.get("AR") else g.relu(g.affine(xn, w1, bb1)), w2, bb2)
        if use_mask:
            y = g.mul(y, g.constant(mask))
        z = g.add(xp, y)
        if final_ln:
            z = g.layer_norm(z, ones2, zeros2)
        out = g.mul(z, g.constant(G))
        loss = g.reduce(M.ReduceOp.Sum, g.reduce(M.ReduceOp.Sum, out, 1), 0, True)
        g.forward(); g.zero_grads(); g.backward(loss)
        rW1, rW2 = ref(use_mask, final_ln)
        e1 = np.linalg.norm(g.param_grad("W1") - rW1) / np.linalg.norm(rW1)
        e2 = np.linalg.norm(g.param_grad("W2") - rW2) / np.linalg.norm(rW2)
        print(f"mask={use_mask} finalLN={final_ln}: dW1 rel {e1:.2e}  dW2 rel {e2:.2e}")
