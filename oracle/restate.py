"""TEST INFRASTRUCTURE ONLY -- a numpy restatement of the reference's
arithmetic on the training path, used to check single kernels.

Each function cites the reference file:line it restates (paths relative to
/root/reference/proj).  The restatement is itself pinned against the
unmodified reference (oracle/_ref via oracle/refbind.py) and the golden
values of the reference's own tests in tests/test_oracle_cpu.py.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU arm may use oracle/.
"""
from __future__ import annotations

import numpy as np

F = np.float32


# ---------------------------------------------------------------- layer norm
def layernorm_fwd(x, g, b, eps=1e-9):
    """layerNormInto, src/tensor.cpp:545-572 (two-pass, population variance)."""
    x = x.astype(np.float64)
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    rs = 1.0 / np.sqrt(var + eps)
    xh = (x - mu) * rs
    return (g * xh + b).astype(F), rs[..., 0].astype(F), xh.astype(F)


def layernorm_bwd(dy, g, rs, xh):
    """layerNormBackward, src/tensor.cpp:574-599."""
    dy = dy.astype(np.float64)
    d = dy.shape[-1]
    dxh = dy * g
    m1 = dxh.sum(-1, keepdims=True) / d
    m2 = (dxh * xh).sum(-1, keepdims=True) / d
    dx = rs[..., None] * (dxh - m1 - xh * m2)
    dg = (dy * xh).reshape(-1, d).sum(0)
    db = dy.reshape(-1, d).sum(0)
    return dx.astype(F), dg.astype(F), db.astype(F)


# ------------------------------------------------------------------ softmax
def softmax_fwd(x, mask=None):
    """softmaxInto, src/tensor.cpp:393-440: masked entries are exactly 0;
    a fully-masked row raises NumericError in the reference."""
    x = x.astype(np.float64)
    m = np.ones_like(x) if mask is None else np.broadcast_to(mask, x.shape) != 0
    if not np.all(m.any(-1)):
        raise FloatingPointError("softmax over a fully-masked row")
    xm = np.where(m, x, -np.inf)
    mx = xm.max(-1, keepdims=True)
    e = np.where(m, np.exp(xm - mx), 0.0)
    return (e / e.sum(-1, keepdims=True)).astype(F)


def softmax_bwd(y, go):
    """graph.cpp:538-553: dx = y * (g - sum(g*y))."""
    y = y.astype(np.float64)
    go = go.astype(np.float64)
    return (y * (go - (go * y).sum(-1, keepdims=True))).astype(F)


# ------------------------------------------------------------ cross-entropy
def xent(logits, targets, mask=None):
    """crossEntropy, src/graph.cpp:859-924: mean over unmasked positions;
    returns (loss, dlogits for an upstream gradient of 1)."""
    V = logits.shape[-1]
    lg = logits.reshape(-1, V).astype(np.float64)
    t = np.asarray(targets).reshape(-1)
    m = np.ones(len(t)) if mask is None else np.asarray(mask, np.float64).reshape(-1)
    mx = lg.max(-1, keepdims=True)
    e = np.exp(lg - mx)
    s = e.sum(-1, keepdims=True)
    p = e / s
    lse = (mx + np.log(s))[:, 0]
    count = m[m != 0].sum()
    if count == 0:
        raise ValueError("cross entropy over a fully-masked batch")
    loss = (m * (lse - lg[np.arange(len(t)), t])).sum() / count
    g = p * (m / count)[:, None]
    g[np.arange(len(t)), t] -= m / count
    return float(loss), g.reshape(logits.shape).astype(F)


# ------------------------------------------------------ multi-head attention
def mha_core(q, k, v, key_mask, causal, heads):
    """MultiHeadAttention::apply core, src/layers.cpp:83-126 (after the
    projections): split heads, scores = (q k^T) * (float)(1/sqrt(dk)), masked
    softmax with the rule j > tk - tq + i for causal (:115-116), context,
    merge heads.  q [b,tq,d], k/v [b,tk,d] -> (out [b,tq,d], probs)."""
    b, tq, d = q.shape
    tk = k.shape[1]
    dk = d // heads
    scale = np.float64(F(1.0 / np.sqrt(dk)))
    qh = q.reshape(b, tq, heads, dk).transpose(0, 2, 1, 3).astype(np.float64)
    kh = k.reshape(b, tk, heads, dk).transpose(0, 2, 1, 3).astype(np.float64)
    vh = v.reshape(b, tk, heads, dk).transpose(0, 2, 1, 3).astype(np.float64)
    s = np.einsum("bhid,bhjd->bhij", qh, kh) * scale
    m = np.ones((b, 1, tq, tk))
    if key_mask is not None:
        m = m * (np.asarray(key_mask)[:, None, None, :] != 0)
    if causal:
        i = np.arange(tq)[:, None]
        j = np.arange(tk)[None, :]
        m = m * (j <= tk - tq + i)
    p = softmax_fwd(s, m).astype(np.float64)
    o = np.einsum("bhij,bhjd->bhid", p, vh)
    return o.transpose(0, 2, 1, 3).reshape(b, tq, d).astype(F), p.astype(F)


def mha_core_bwd(q, k, v, p, go, heads):
    """Backward of mha_core through the reference's node chain (dot, scale,
    softmax, dot: graph.cpp:293-332, 236-252, 538-553)."""
    b, tq, d = q.shape
    tk = k.shape[1]
    dk = d // heads
    scale = np.float64(F(1.0 / np.sqrt(dk)))
    sp = lambda x, t: x.reshape(b, t, heads, dk).transpose(0, 2, 1, 3).astype(np.float64)
    qh, kh, vh, goh = sp(q, tq), sp(k, tk), sp(v, tk), sp(go, tq)
    p = p.astype(np.float64)
    dv = np.einsum("bhij,bhid->bhjd", p, goh)
    dp = np.einsum("bhid,bhjd->bhij", goh, vh)
    ds = p * (dp - (dp * p).sum(-1, keepdims=True)) * scale
    dq = np.einsum("bhij,bhjd->bhid", ds, kh)
    dkk = np.einsum("bhij,bhid->bhjd", ds, qh)
    mg = lambda x, t: x.transpose(0, 2, 1, 3).reshape(b, t, d).astype(F)
    return mg(dq, tq), mg(dkk, tk), mg(dv, tk)


# ------------------------------------------------------------------ GRU cell
def gru_fwd(h, x, W, ln=False, eps=1e-9):
    """gruCell forward, src/graph.cpp:692-746 with gruPre :633-645.
    W: dict Uz,Ur,Uh,bz,br,bh[,Wz,Wr,Wx][,lnGz,lnBz,lnGr,lnBr[,lnGx,lnBx]]."""
    h = h.astype(np.float64)
    sig = lambda a: 1.0 / (1.0 + np.exp(-a))
    lnf = (lambda a, g, bb: layernorm_fwd(a, W[g], W[bb], eps)[0].astype(np.float64)) if ln \
        else (lambda a, g, bb: a)
    pre_z = h @ W["Uz"] + (x @ W["Wz"] if x is not None else 0) + W["bz"]
    pre_r = h @ W["Ur"] + (x @ W["Wr"] if x is not None else 0) + W["br"]
    z = sig(lnf(pre_z, "lnGz", "lnBz"))
    r = sig(lnf(pre_r, "lnGr", "lnBr"))
    uh = h @ W["Uh"]
    ac = lnf(x @ W["Wx"], "lnGx", "lnBx") if x is not None else 0.0
    ht = np.tanh(ac + (r * uh + W["bh"]))
    return ((1 - z) * ht + z * h).astype(F)


# --------------------------------------------------------------- optimizer
def adam_step(theta, grad, m, v, lr, step, b1=0.9, b2=0.999, eps=1e-8):
    """Adam::updateTensor, src/train.cpp:30-47 (float32 arithmetic, bias
    corrections computed in double and cast)."""
    theta, grad, m, v = (np.asarray(a, F).copy() for a in (theta, grad, m, v))
    b1, b2, eps, lr = F(b1), F(b2), F(eps), F(lr)
    c1 = F(1.0 - np.power(np.float64(b1), step))
    c2 = F(1.0 - np.power(np.float64(b2), step))
    m = b1 * m + (F(1) - b1) * grad
    v = b2 * v + (F(1) - b2) * grad * grad
    mh = m / c1
    vh = v / c2
    theta = theta - lr * mh / (np.sqrt(vh).astype(F) + eps)
    return theta, m, v


def ema(avg, theta, beta=0.9999):
    """AveragedParameters::update, src/train.cpp:69-79."""
    beta = F(beta)
    return (beta * np.asarray(avg, F) + (F(1) - beta) * np.asarray(theta, F)).astype(F)


def lr_schedule(step, base=3e-4, warmup=16000):
    """LrSchedule::operator(), src/train.cpp:61-67."""
    base = F(base)
    if step <= warmup:
        return F(base * F(step) / F(warmup))
    return F(base * F(np.sqrt(warmup / step)))


# --------------------------------------------------------- data parallelism
def fnv1a(s: str) -> int:
    """hash64, include/mtk/common.h:41-48."""
    h = 1469598103934665603
    for c in s.encode():
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def mix_seed(seed: int, update: int, worker: int) -> int:
    """mixSeed, src/train.cpp:170-176 (uint64 wrap-around)."""
    M = 0xFFFFFFFFFFFFFFFF
    h = fnv1a("update")
    h ^= (seed + 0x9E3779B97F4A7C15 + ((h << 6) & M) + (h >> 2)) & M
    h ^= (update * 0xBF58476D1CE4E5B9) & M
    h ^= ((worker + 1) * 0x94D049BB133111EB) & M
    return h & M


def dp_combine(grads, tokens):
    """trainSync's worker-ordered weighted combine, src/train.cpp:254-269:
    g = g0*(t0/T), then g += (ti/T)*gi for i >= 1 (float32)."""
    total = F(sum(F(t) for t in tokens))
    g = np.asarray(grads[0], F) * (F(tokens[0]) / total)
    for gi, ti in zip(grads[1:], tokens[1:]):
        g = g + (F(ti) / total) * np.asarray(gi, F)
    return g


def shard(take: int, world: int, local_workers: int, rank: int):
    """Worker indices rank `rank` runs in one update of `take` batches when
    `world` ranks each run `local_workers` of the reference's workers
    (worker i = rank*L + j handles batches[idx + i], train.cpp:232)."""
    return [rank * local_workers + j for j in range(local_workers)
            if rank * local_workers + j < take]
