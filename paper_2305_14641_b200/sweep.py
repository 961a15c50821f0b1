"""Sigma grids and mutation detection (host logic of the sweep driver).

Mirrors proj/src/sweep.cpp:11-71 operation for operation (Python floats are
IEEE doubles and math.exp / math.log are the C library's exp / log, so the
grids are the same bits as the reference's std::exp(lo + (hi - lo) * k /
(steps - 1))).
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple


def log_sigma_grid(default_distance: float, steps: int = 30, lo_factor: float = 0.1,
                   hi_factor: float = 3.0) -> List[float]:
    """sweep.cpp:11-26."""
    if default_distance <= 0.0 or lo_factor <= 0.0 or hi_factor <= lo_factor:
        raise ValueError("invalid sigma grid bounds")
    if steps < 1:
        raise ValueError("sigma grid needs at least one point")
    lo = math.log(lo_factor * default_distance)
    hi = math.log(hi_factor * default_distance)
    if steps == 1:
        return [math.exp(lo)]
    return [math.exp(lo + (hi - lo) * k / (steps - 1)) for k in range(steps)]


def linear_sigma_grid(lo: float, hi: float, steps: int) -> List[float]:
    """sweep.cpp:28-38."""
    if lo <= 0.0 or hi < lo:
        raise ValueError("invalid sigma grid bounds")
    if steps < 1:
        raise ValueError("sigma grid needs at least one point")
    if steps == 1:
        return [lo]
    return [lo + (hi - lo) * k / (steps - 1) for k in range(steps)]


def check_grid(sigmas: Sequence[float]):
    """run_sweep's validation (sweep.cpp:42-47)."""
    if len(sigmas) == 0:
        raise ValueError("sigma grid is empty")
    for k, s in enumerate(sigmas):
        if not (s > 0.0):
            raise ValueError("sigma must be positive")
        if k > 0 and s <= sigmas[k - 1]:
            raise ValueError("sigma grid must be strictly ascending")


def detect_mutation(sigmas: Sequence[float], counts: Sequence[int]) -> Optional[Tuple[float, float, int]]:
    """sweep.cpp:61-71: the consecutive pair with the largest cluster-count
    drop, earliest on ties; None if the count never decreases."""
    if len(counts) < 2:
        raise ValueError("mutation detection needs at least two records")
    best = None
    for k in range(len(counts) - 1):
        drop = counts[k] - counts[k + 1]
        if drop >= 1 and (best is None or drop > best[2]):
            best = (sigmas[k], sigmas[k + 1], drop)
    return best
