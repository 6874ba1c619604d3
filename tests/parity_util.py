"""Shared gradient / parameter parity checks against the reference oracle.

Per-tensor bounds:  ||g - g_ref||_2 <= tol * ||g_ref||_2 for
every parameter tensor, tol = 1e-4 in FP32 mode and 1e-2 in TF32 mode.  The
only absolute floor is for tensors whose exact gradient is zero (attention
key biases: softmax is invariant to a per-row shift, so dL/dkB = 0 and the
reference's value is rounding noise); those are recognised by
||g_ref|| <= ZERO_REL * ||G_ref|| and must satisfy ||g - g_ref|| <= ZERO_REL * ||G_ref||.
"""
from __future__ import annotations

import json
import os

import numpy as np

GRAD_TOL = {"fp32": 1e-4, "tf32": 1e-2}
ZERO_REL = 1e-5


def grad_ratios(names, mine, ref):
    """[(name, ||d||, ||g_ref||, ratio, zero_grad)] with ratio = ||d|| / bound-scale."""
    G = np.sqrt(sum(float(np.sum(ref[n].astype(np.float64) ** 2)) for n in names))
    out = []
    for n in names:
        a = np.asarray(mine[n], np.float64)
        b = np.asarray(ref[n], np.float64)
        d = float(np.linalg.norm(a - b))
        nb = float(np.linalg.norm(b))
        zero = nb <= ZERO_REL * G
        scale = ZERO_REL * G if zero else nb
        out.append((n, d, nb, d / scale if scale > 0 else (0.0 if d == 0 else np.inf), zero))
    return out, G


def check_grads(names, mine, ref, prec, label):
    """Assert the per-tensor bound; returns the worst ratio d / (tol * ||g_ref||)."""
    tol = GRAD_TOL[prec]
    rows, G = grad_ratios(names, mine, ref)
    worst = max(rows, key=lambda r: r[3] / (1.0 if r[4] else tol))
    rep = {"label": label, "prec": prec, "tol": tol, "G": G,
           "worst": {"name": worst[0], "rel": worst[3], "zero_grad": worst[4]},
           "rel": {r[0]: r[3] for r in rows}}
    d = os.environ.get("MTK_PARITY_DUMP")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"{label}_{prec}.json"), "w") as f:
            json.dump(rep, f, indent=1)
    print(f"[parity] {label} {prec}: worst {worst[0]} rel {worst[3]:.3e} (tol {tol:g})")
    bad = [(r[0], r[3]) for r in rows if r[3] > (1.0 if r[4] else tol)]
    assert not bad, f"{label} {prec}: {len(bad)} tensors over the bound: {bad[:8]}"
    return worst[3] / (1.0 if worst[4] else tol)


def check_adam_fp32(names, after_mine, after_ref, lr, frac=1e-3):
    """Parameters after one Adam step, FP32 mode: |d| <= 1e-3 lr for >= 99.9 %
    of elements and <= 2 lr everywhere (step 1 moves each element by about
    lr*sign(g); elements whose |g| is near eps flip on rounding noise)."""
    bad = total = 0
    for n in names:
        d = np.abs(np.asarray(after_mine[n], np.float64) - np.asarray(after_ref[n], np.float64))
        bad += int(np.sum(d > 1e-3 * lr))
        total += d.size
        assert np.all(d <= 2.0 * lr + 1e-7 * np.abs(after_ref[n])), n
    assert bad <= frac * total, (bad, total)


def check_adam_sign(names, before, after_mine, after_ref, grads_ref, min_agree=0.99):
    """TF32 mode: the first Adam step moves each parameter by ~ -lr*sign(g);
    over elements whose reference gradient is not negligible
    (|g| > 1e-3 * rms of its tensor) the step's sign must agree with the
    reference's for >= min_agree of them, and no step may exceed 2 lr."""
    agree = total = 0
    for n in names:
        g = np.asarray(grads_ref[n], np.float64)
        rms = np.sqrt(np.mean(g * g)) if g.size else 0.0
        sel = np.abs(g) > 1e-3 * rms
        dm = (np.asarray(after_mine[n], np.float64) - before[n])[sel]
        dr = (np.asarray(after_ref[n], np.float64) - before[n])[sel]
        agree += int(np.sum(np.sign(dm) == np.sign(dr)))
        total += int(sel.sum())
    frac = agree / max(total, 1)
    print(f"[parity] adam sign agreement {frac:.6f} over {total} elements")
    assert frac >= min_agree, frac
    return frac
