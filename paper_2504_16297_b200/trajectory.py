"""Outcome selection shared by the pre-trajectory samplers.

Only ``select_index`` (ref ``pkg/src/trajsim/trajectory.py:27-37``) is on the
PTSBE path: the PTS strategies draw each site's Kraus outcome with it.  The
conventional Algorithm-1 simulator in the same reference module is the
baseline the paper accelerates and is out of scope for this engine (SURVEY
section 2, row 7).
"""

from __future__ import annotations

import numpy as np

from .errors import ValidationError


def select_index(r: float, probs) -> int:
    """Smallest k whose running sum of probs exceeds r; the last index if none does.

    The running sum is accumulated left to right in float64 -- the same
    rounding as ``np.cumsum`` -- so vectorised callers can use
    ``searchsorted(cumsum(probs), r, side="right")`` and stay bit-exact.
    """
    n = len(probs)
    if n == 0:
        raise ValidationError("empty probability list")
    running = 0.0
    for k, p in enumerate(probs):
        running += p
        if r < running:
            return k
    return n - 1


def select_indices(r: np.ndarray, probs) -> np.ndarray:
    """Vectorised ``select_index`` over an array of uniforms (bit-identical)."""
    edges = np.cumsum(np.asarray(probs, dtype=np.float64))
    k = np.searchsorted(edges, r, side="right")
    return np.minimum(k, len(edges) - 1)
