"""Host-side numeric constants for the kernels, rounded as numpy rounds them.

sqrt_le_bound(t) / sqrt_lt_bound(t): the largest float32 x >= 0 with
fl(sqrt(x)) <= t (resp. < t).  float32 sqrt is correctly rounded on both
sides (numpy's np.sqrt and CUDA's __fsqrt_rn) and monotonic, so for every
float32 d2 >= 0

    fl(sqrt(d2)) <= t   <=>   d2 <= sqrt_le_bound(t)

which lets a kernel decide "within range" from the squared distance alone
and take the square root only where the distance itself is needed (an
active contact, a reward term).  Decisions stay bit-identical to the
reference's `norm(...) <= t` (dynamics.py:57, common.py:53-58, ...).
"""
from __future__ import annotations

import numpy as np

F32 = np.float32


def _sqrt(x) -> np.float32:
    return np.sqrt(F32(x), dtype=F32)


def sqrt_le_bound(t) -> np.float32:
    """Largest float32 x >= 0 with sqrt(x) <= t (float32)."""
    t = F32(t)
    if not t >= 0:
        return F32(-1.0)          # nothing qualifies (callers compare d2 <= bound)
    if np.isinf(t):
        return F32(np.inf)
    x = F32(t * t)
    inf = F32(np.inf)
    while _sqrt(x) > t:
        x = np.nextafter(x, F32(0), dtype=F32)
    while True:
        nx = np.nextafter(x, inf, dtype=F32)
        if _sqrt(nx) <= t:
            x = nx
        else:
            return x


def sqrt_lt_bound(t) -> np.float32:
    """Largest float32 x >= 0 with sqrt(x) < t (float32); -1 if none."""
    t = F32(t)
    if not t > 0:
        return F32(-1.0)
    prev = np.nextafter(t, F32(0), dtype=F32)
    return sqrt_le_bound(prev)
