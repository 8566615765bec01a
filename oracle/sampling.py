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


def render_dictionary_atlas(atoms: np.ndarray, pi: np.ndarray, patch_shape) -> np.ndarray:
    """server.py:84-120: atoms min-max normalised (constant -> 0.5), ordered by
    descending pi (stable), tiled into a ceil(sqrt(K)) grid with mid-grey
    1-pixel separators and empty cells."""
    import math

    shape = tuple(int(b) for b in patch_shape)
    k = atoms.shape[0]
    a = np.asarray(atoms, dtype=np.float64).reshape((k,) + shape)
    if len(shape) == 3:
        a = a[:, :, :, 0]
    elif len(shape) == 1:
        a = a[:, None, :]
    elif len(shape) != 2:
        raise ValueError(f"cannot render atlas for patch rank {len(shape)}")
    b0, b1 = a.shape[1], a.shape[2]
    lo = a.min(axis=(1, 2), keepdims=True)
    hi = a.max(axis=(1, 2), keepdims=True)
    span = hi - lo
    flat = span[:, 0, 0] == 0
    with np.errstate(invalid="ignore", divide="ignore"):
        tiles = (a - lo) / span
    tiles[flat] = 0.5
    order = np.argsort(-np.asarray(pi), kind="stable")
    grid = math.ceil(math.sqrt(k))
    canvas = np.full((grid * b0 + grid - 1, grid * b1 + grid - 1), 0.5, dtype=np.float64)
    for slot, idx in enumerate(order):
        r, c = divmod(slot, grid)
        canvas[r * (b0 + 1):r * (b0 + 1) + b0, c * (b1 + 1):c * (b1 + 1) + b1] = tiles[idx]
    return canvas
