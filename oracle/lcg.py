"""Vectorised restatement of the reference weight stream (TEST ONLY).

Reference: `/root/reference/pkg/src/treepipe/model.py:28-44`
(``lcg_uniform_stream``): state' = state*6364136223846793005 +
1442695040888963407 (mod 2^64), sample = (state >> 11) / 2^53, then the
whole array is mapped with ``* 0.2 - 0.1`` (two separately rounded f64
ops).  Here the states are produced by affine jump-ahead on uint64 arrays
(numpy wraps mod 2^64), which is bit-identical to the scalar loop.
"""

from __future__ import annotations

import numpy as np

MUL = 6364136223846793005
INC = 1442695040888963407
MASK = (1 << 64) - 1


def affine_power(steps: int) -> tuple[int, int]:
    """(a, c) with s_{i+steps} = a*s_i + c mod 2^64."""
    a, c = 1, 0  # identity map
    base_a, base_c = MUL, INC
    while steps:
        if steps & 1:
            a, c = (base_a * a) & MASK, (base_a * c + base_c) & MASK
        base_a, base_c = (base_a * base_a) & MASK, (base_a * base_c + base_c) & MASK
        steps >>= 1
    return a, c


def lcg_states(seed: int, count: int, start: int = 0) -> np.ndarray:
    """States s_{start+1} .. s_{start+count} of the stream seeded with ``seed``."""
    out = np.empty(count, dtype=np.uint64)
    if count == 0:
        return out
    a0, c0 = affine_power(start + 1)
    first = (a0 * (seed & MASK) + c0) & MASK
    head = min(count, 1024)
    s = first
    for i in range(head):
        out[i] = s
        s = (s * MUL + INC) & MASK
    filled = head
    with np.errstate(over="ignore"):
        while filled < count:
            n = min(filled, count - filled)
            a, c = affine_power(filled)
            out[filled : filled + n] = out[:n] * np.uint64(a) + np.uint64(c)
            filled += n
    return out


def uniform_stream(seed: int, count: int, start: int = 0) -> np.ndarray:
    """float64 samples in [-0.1, 0.1), bit-identical to the reference."""
    u = (lcg_states(seed, count, start) >> np.uint64(11)).astype(np.float64) / float(1 << 53)
    return u * 0.2 - 0.1
