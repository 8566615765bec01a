"""Host-side input generators: synthetic frames and sampling masks.

These are hot-path *inputs*, not the hot path (SURVEY.md §2 rows 6 and 8 are
out of scope for acceleration).  They restate the reference generators so both
arms of every measurement see identical bytes:

* ``synthetic_texture`` — reference pkg/src/patchbeam/sources.py:118-141
  (seeded sum of 8 sinusoidal gratings, normalized to [0, 1]);
  ``synthetic_frames`` — SyntheticSource.read_item (sources.py:95-115, phase 0.15·t).
* ``make_mask`` — reference pkg/src/patchbeam/sampling.py: exact budget
  floor(r·M + 0.5) (53-56); ``uniform-random`` (69-74), ``line-hop`` (132-164),
  ``explicit-list`` (167-174).  Keys (seed, DOMAIN_MASK, strategy id) (59-60).
* ``stem_lattice`` — a seeded STEM-like frame (Gaussian atomic columns on a
  slightly distorted lattice plus Poisson shot noise), new in this repo, used
  for the "EM-like" bench inputs.
"""

from __future__ import annotations

import numpy as np

from .rng import DOMAIN_MASK, DOMAIN_SYNTH, keyed_rng

_STRATEGY_IDS = {"uniform-random": 1, "stratified": 2, "line-hop": 3,
                 "explicit-list": 4, "adaptive-residual": 5}


def synthetic_texture(shape, seed=0, gratings=8, phase=0.0):
    rng = keyed_rng(seed, DOMAIN_SYNTH)
    h, w = shape
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    yy /= h
    xx /= w
    img = np.zeros(shape, dtype=np.float64)
    for _ in range(gratings):
        amp = rng.uniform(0.3, 1.0)
        fy, fx = rng.uniform(1.0, 12.0, size=2)
        phi = rng.uniform(0.0, 2.0 * np.pi)
        img += amp * np.sin(2.0 * np.pi * (fy * yy + fx * xx) + phi + phase)
    lo, hi = img.min(), img.max()
    return (img - lo) / (hi - lo) if hi > lo else np.zeros(shape, dtype=np.float64)


def synthetic_frames(shape, count, seed=0):
    return [synthetic_texture(shape, seed=seed, phase=0.15 * t) for t in range(count)]


def stem_lattice(shape, seed=0, spacing=7.5, sigma=1.4, dose=200.0):
    """EM-like 2-D frame: Gaussian columns on a lattice + Poisson noise, in [0, 1]."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=int(seed), spawn_key=(11,)))
    h, w = shape
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    img = np.zeros(shape)
    theta = 0.21
    ax = np.array([np.cos(theta), np.sin(theta)]) * spacing
    ay = np.array([-np.sin(theta), np.cos(theta)]) * spacing
    n = int(max(h, w) / spacing) + 4
    for a in range(-n, 2 * n):
        for b in range(-n, 2 * n):
            cy, cx = a * ax[0] + b * ay[0], a * ax[1] + b * ay[1]
            if -3 * sigma <= cy < h + 3 * sigma and -3 * sigma <= cx < w + 3 * sigma:
                z = 0.6 + 0.4 * ((a + b) % 2)
                y0, y1 = int(max(0, cy - 4 * sigma)), int(min(h, cy + 4 * sigma + 1))
                x0, x1 = int(max(0, cx - 4 * sigma)), int(min(w, cx + 4 * sigma + 1))
                if y0 < y1 and x0 < x1:
                    img[y0:y1, x0:x1] += z * np.exp(
                        -((yy[y0:y1, x0:x1] - cy) ** 2 + (xx[y0:y1, x0:x1] - cx) ** 2) / (2 * sigma ** 2))
    img = rng.poisson(img * dose) / dose
    lo, hi = img.min(), img.max()
    return (img - lo) / (hi - lo) if hi > lo else np.zeros(shape)


def sample_budget(ratio, shape):
    return int(np.floor(ratio * int(np.prod(shape)) + 0.5))


def _mask_rng(seed, kind, *sub):
    return keyed_rng(seed, DOMAIN_MASK, _STRATEGY_IDS[kind], *sub)


def make_mask(shape, ratio, kind="uniform-random", seed=0, indices=()):
    shape = tuple(int(m) for m in shape)
    total = int(np.prod(shape))
    flat = np.zeros(total, dtype=bool)
    if kind == "uniform-random":
        picks = _mask_rng(seed, kind).choice(total, size=sample_budget(ratio, shape), replace=False)
        flat[picks] = True
        return flat.reshape(shape)
    if kind == "explicit-list":
        idx = np.asarray(indices, dtype=np.int64)
        flat[idx] = True
        return flat.reshape(shape)
    if kind == "line-hop":
        if not 2 <= len(shape) <= 3:
            raise ValueError("line-hop supports 2D/3D shapes only")
        row_len = shape[-1]
        n_rows = total // row_len
        n_full, partial = divmod(sample_budget(ratio, shape), row_len)
        n_lines = n_full + (1 if partial else 0)
        rng = _mask_rng(seed, kind)
        m = np.zeros((n_rows, row_len), dtype=bool)
        if n_lines:
            edges = np.linspace(0, n_rows, n_lines + 1)
            rows = []
            for j in range(n_lines):
                lo = int(edges[j])
                hi = max(int(edges[j + 1]), lo + 1)
                rows.append(lo + int(rng.integers(0, hi - lo)))
            rows = np.unique(np.asarray(rows, dtype=np.int64))
            while rows.size < n_lines:
                free = np.setdiff1d(np.arange(n_rows), rows)
                rows = np.sort(np.append(rows, free[: n_lines - rows.size]))
            m[rows[:n_full], :] = True
            if partial:
                ph = int(rng.integers(0, row_len))
                m[rows[n_full], (ph + np.arange(partial)) % row_len] = True
        return m.reshape(shape)
    raise ValueError(f"unsupported mask kind {kind!r}")
