"""CPU restatement (TEST INFRASTRUCTURE ONLY) of the live path's tail: the uint8
wire panels, the residual map that drives adaptive sampling, and the exploit
half of the adaptive-residual sampler.  Only tests/ may import this module.

Pinned by tests/golden/live_tail.npz, produced by running the reference itself
(tests/golden/make_golden.py live_tail).
"""

from __future__ import annotations

import numpy as np


def quantize_panel(panel: np.ndarray) -> np.ndarray:
    """server.py:46-53: rank-3 panels show slice 0; round(clip(x, 0, 1) * 255)."""
    panel = np.asarray(panel)
    if panel.ndim == 3:
        panel = panel[:, :, 0]
    if panel.ndim != 2:
        raise ValueError(f"wire panels must be 2D, got rank {panel.ndim}")
    return np.round(np.clip(panel, 0.0, 1.0) * 255.0).astype(np.uint8)


def residual_map(recon: np.ndarray, prev: np.ndarray | None) -> np.ndarray:
    """pipeline.py:265-269: (recon - prev)^2, zeros for the first frame."""
    if prev is None:
        return np.zeros_like(recon)
    d = recon - prev
    return d * d


def sample_budget(ratio: float, total: int) -> int:
    """sampling.py:53-56: round-half-up of ratio * total."""
    return int(np.floor(ratio * total + 0.5))


def adaptive_split(ratio: float, exploit_fraction: float, total: int) -> tuple[int, int]:
    """sampling.py:193-197: (budget, n_exploit)."""
    budget = sample_budget(ratio, total)
    n_exploit = int(np.floor(exploit_fraction * budget + 0.5))
    return budget, min(max(n_exploit, 0), budget)


def adaptive_exploit(residual: np.ndarray, ratio: float, exploit_fraction: float) -> np.ndarray:
    """sampling.py:199-201: flat indices of the n_exploit largest residuals, ties
    broken by the lowest flat index (stable argsort of -residual)."""
    r = np.asarray(residual, dtype=np.float64).ravel()
    _, n_exploit = adaptive_split(ratio, exploit_fraction, r.size)
    return np.argsort(-r, kind="stable")[:n_exploit]
