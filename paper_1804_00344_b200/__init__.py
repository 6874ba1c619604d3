"""B200-native rebuild of the Marian/mtk encoder-decoder training step.

The C++ host framework (ExpressionGraph, layers, models, batching, Adam/EMA,
synchronous data-parallel trainer) lives in libmtkhost.so and is exposed as
the `_mtk` extension; every arithmetic op runs in the sm_100a kernels of
libmtkcuda.so behind the C-ABI in include/mtk_cuda.h.  There is no CPU
fallback: importing this package without the built libraries fails.
"""
from __future__ import annotations

import os

_HERE = os.path.dirname(os.path.abspath(__file__))


def _load():
    try:
        from . import _mtk  # noqa: F401
    except ImportError as e:  # pragma: no cover - fails loudly by design
        raise ImportError(
            "paper_1804_00344_b200: native libraries are not built "
            "(run __graft_entry__.build()); there is no CPU fallback") from e
    return _mtk


mtk = _load()


def native_libraries():
    """Paths of the in-tree native libraries this package runs on."""
    return [os.path.join(_HERE, n) for n in ("libmtkcuda.so", "libmtkhost.so")]


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
