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


from .configs import CONFIGS, TOKEN_BUDGET, algorithmic_flops, config_text  # noqa: E402,F401
