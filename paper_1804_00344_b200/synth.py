"""Synthetic parallel corpus used by every benchmark and parity config.

Specification: SURVEY.md §8(d) ("Synthetic data generator (all configs)").
Pair i has source length 16 + splitmix64(1234*1000003 + i) mod 17 and target
length 16 + splitmix64(5678*1000003 + i) mod 17 (16..32 tokens before the
</s> that batching appends, data.cpp:149-166); token j of the source is
2 + splitmix64((i << 20) ^ j ^ 0xabc) mod (V - 2), targets use 0xdef.  Ids are
uniform over [2, V): 0 is </s> and 1 is <unk> (data.h:14-15).
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def pair_lengths(n: int, start: int = 0):
    i = np.arange(start, start + n, dtype=np.uint64)
    ls = 16 + (splitmix64(np.uint64(1234 * 1000003) + i) % np.uint64(17)).astype(np.int64)
    lt = 16 + (splitmix64(np.uint64(5678 * 1000003) + i) % np.uint64(17)).astype(np.int64)
    return ls, lt


def _tokens(i: int, n: int, salt: int, vocab: int):
    j = np.arange(n, dtype=np.uint64)
    x = (np.uint64(i) << np.uint64(20)) ^ j ^ np.uint64(salt)
    return (2 + (splitmix64(x) % np.uint64(vocab - 2))).astype(np.int32)


def corpus(n: int, vocab: int, start: int = 0):
    """Returns (sources, targets): lists of int32 arrays without </s>."""
    ls, lt = pair_lengths(n, start)
    src = [_tokens(start + k, int(ls[k]), 0xABC, vocab) for k in range(n)]
    tgt = [_tokens(start + k, int(lt[k]), 0xDEF, vocab) for k in range(n)]
    return src, tgt
