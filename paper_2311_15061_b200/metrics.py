"""Image-quality metrics used as the parity metric (host side).

``psnr``/``mse`` restate reference pkg/src/patchbeam/metrics.py:26-40.  The
reference has no SSIM; ``ssim`` here is the standard
Wang et al. 2004 index (Gaussian window sigma=1.5, truncated at 3.5 sigma,
K1=0.01, K2=0.03, data range 1, mean over the valid interior), computed
identically on both implementations' outputs by the harness.
"""

from __future__ import annotations

import math

import numpy as np


def mse(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    d = a - b
    return float(np.mean(d * d))


def psnr(a, b, peak: float = 1.0) -> float:
    if peak <= 0:
        raise ValueError("peak must be > 0")
    e = mse(a, b)
    return math.inf if e == 0.0 else 10.0 * math.log10(peak * peak / e)


def ssim(a, b, data_range: float = 1.0, sigma: float = 1.5) -> float:
    from scipy.ndimage import gaussian_filter

    x = np.asarray(a, dtype=np.float64)
    y = np.asarray(b, dtype=np.float64)
    if x.shape != y.shape:
        raise ValueError("shape mismatch")
    f = lambda z: gaussian_filter(z, sigma, truncate=3.5, mode="reflect")  # noqa: E731
    mx, my = f(x), f(y)
    vx = f(x * x) - mx * mx
    vy = f(y * y) - my * my
    cxy = f(x * y) - mx * my
    c1, c2 = (0.01 * data_range) ** 2, (0.03 * data_range) ** 2
    s = ((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2))
    r = int(3.5 * sigma + 0.5)
    if all(n > 2 * r for n in s.shape):
        s = s[tuple(slice(r, -r) for _ in s.shape)]
    return float(s.mean())
