"""The BASELINE.json configurations, ModelConfig text, and the SURVEY.md 8(d)
algorithmic FLOP count of a training step.  Pure Python (no native
libraries): bench.py's reference arm loads this file by path so that arm never
maps the product's .so files.
"""
from __future__ import annotations

import numpy as np


def config_text(arch="transformer", vocab=32000, emb=512, state=1024, heads=8, layers=6,
                dropout=0.0, tying="all", layer_norm=False, post_norm=False):
    """ModelConfig text (models.cpp:12-30 key order)."""
    return (f"architecture: {arch}\nsource-vocab: {vocab}\ntarget-vocab: {vocab}\n"
            f"emb-dim: {emb}\nstate-dim: {state}\nheads: {heads}\nlayers: {layers}\n"
            f"dropout: {dropout}\ntying: {tying}\nlayer-norm: {int(layer_norm)}\n"
            f"post-norm: {int(post_norm)}\n")


# The five BASELINE.json configurations.
CONFIGS = {
    "tiny": dict(arch="transformer", vocab=8000, emb=256, heads=4, layers=2),
    "shallow": dict(arch="s2s-shallow", vocab=50000, emb=512, state=1024),
    "deep": dict(arch="s2s-deep", vocab=50000, emb=512, state=1024, layer_norm=True),
    "base": dict(arch="transformer", vocab=32000, emb=512, heads=8, layers=6),
    "big": dict(arch="transformer", vocab=32000, emb=1024, heads=16, layers=6),
}
TOKEN_BUDGET = {"tiny": 64 * 66, "shallow": 4096, "deep": 4096, "base": 16384, "big": 32768}


def algorithmic_flops(config: str, src_lens, tgt_lens, spec=None):
    """SURVEY.md 8(d) algorithmic FLOPs of one training step (3x forward) over
    REAL tokens: src_lens / tgt_lens are the per-sentence unmasked lengths
    (incl. </s>).  Returns {"gemm": dense-contraction FLOPs, "attention":
    attention-core FLOPs, "total": sum}.

    Transformer: 6*(N_src*c_src + N_tgt*c_tgt) + 6*sum_i(2*L_e*s_i^2*d +
    L_d*(2*t_i^2*d + 2*t_i*s_i*d)), c_src = 12 L_e d^2 + 2 L_d d^2,
    c_tgt = 14 L_d d^2 + d V.  RNN (keys projection hoisted): shallow
    c_src = 6ed + 8d^2, c_tgt = 6ed + 13d^2 + e^2 + eV; deep c_src = 6ed + 26d^2,
    c_tgt = 6ed + 31d^2 + e^2 + eV; attention 6*sum_i 3 t_i s_i d."""
    spec = spec or CONFIGS[config]
    s = np.asarray(src_lens, np.float64)
    t = np.asarray(tgt_lens, np.float64)
    ns, nt = float(s.sum()), float(t.sum())
    V = spec["vocab"]
    if spec["arch"] == "transformer":
        d, L = spec["emb"], spec.get("layers", 6)
        c_src = 12 * L * d * d + 2 * L * d * d
        c_tgt = 14 * L * d * d + d * V
        att = 6 * float(np.sum(2 * L * s * s * d + L * (2 * t * t * d + 2 * t * s * d)))
    else:
        e, d = spec["emb"], spec.get("state", 1024)
        if spec["arch"] == "s2s-shallow":
            c_src, c_tgt = 6 * e * d + 8 * d * d, 6 * e * d + 13 * d * d + e * e + e * V
        else:
            c_src, c_tgt = 6 * e * d + 26 * d * d, 6 * e * d + 31 * d * d + e * e + e * V
        att = 6 * float(np.sum(3 * t * s * d))
    gemm = 6.0 * (ns * c_src + nt * c_tgt)
    return {"gemm": gemm, "attention": att, "total": gemm + att}
