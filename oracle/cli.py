"""ORACLE (test infrastructure only): the CLI entry steps.

Restates reference pkg/src/patchbeam/cli.py:195-212 (_normalize_observed);
pinned against tests/golden/entry.npz (produced by the reference itself).
"""

from __future__ import annotations

import numpy as np


def normalize_observed(frame, mask):
    """cli.py:195-212."""
    vals = frame[mask]
    if vals.size == 0:
        return frame, 1.0, 0.0
    lo, hi = float(vals.min()), float(vals.max())
    if 0.0 <= lo and hi <= 1.0:
        return frame, 1.0, 0.0
    if hi == lo:
        return np.where(mask, 0.0, frame), 1.0, lo
    return (frame - lo) / (hi - lo), hi - lo, lo
