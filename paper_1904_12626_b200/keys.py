"""Host mirror of the packed (score, index) keys the join min-reduces.

Device format (csrc/mpgpu_kernels.cuh mk_key): key = (bits(score) & ~mask) | idx
with score = 1 - corr = d^2 / (2m) >= 0 and mask = 2^b - 1, b = ceil(log2(max
profile length)). Non-negative doubles order like int64, so an elementwise
int64 MIN is an exact min-with-argmin whose ties go to the smallest index —
the merge_min rule (profile.hpp:66-68: ties keep the first, lowest source).
The empty key is INT64_MAX.
"""
from __future__ import annotations

import math

import numpy as np

KEY_NONE = np.int64(0x7FFFFFFFFFFFFFFF)


def index_bits(len_a: int, len_b: int = 0) -> int:
    n = max(int(len_a), int(len_b), 1)
    return max(1, math.ceil(math.log2(n))) if n > 1 else 1


def pack(corr, idx, bits: int) -> np.ndarray:
    """Keys for correlations `corr` with neighbour indices `idx`."""
    s = np.maximum(1.0 - np.asarray(corr, dtype=np.float64), 0.0)
    mask = np.int64((1 << bits) - 1)
    return (s.view(np.int64) & ~mask) | np.asarray(idx, dtype=np.int64)


def pack_score(score, idx, bits: int) -> np.ndarray:
    s = np.asarray(score, dtype=np.float64)
    mask = np.int64((1 << bits) - 1)
    return (s.view(np.int64) & ~mask) | np.asarray(idx, dtype=np.int64)


def unpack(keys, bits: int):
    """(score lower bound, index) per key; index -1 and score inf for KEY_NONE."""
    k = np.asarray(keys, dtype=np.int64)
    mask = np.int64((1 << bits) - 1)
    none = k == KEY_NONE
    idx = np.where(none, -1, k & mask)
    score = np.where(none, np.inf, (k & ~mask).view(np.float64))
    return score, idx
