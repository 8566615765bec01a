"""ORACLE (test infrastructure only): N-D patch gather / overlap-average.

Restates reference pkg/src/patchbeam/patches.py.  The implementation is an
explicit flat-index gather (not the reference's sliding-window view) but every
floating-point operation is the same numpy op on the same operands in the same
order, so outputs are bit-identical:

* grid: origins along dim i are 0, s_i, 2 s_i, ... while o + B_i <= M_i
  (patches.py:64-70, 107-113); patch order is row-major over the grid, element
  order row-major within the patch (patches.py:116-122).
* extract: values = x*o; optional observed-only mean, values = (values-mean)*o
  (patches.py:143-154).
* reconstitute: per-element sum of (estimate + mean) over covering patches in
  ascending (patch, offset) order, divided by coverage; uncovered -> 0 or
  CoverageError (patches.py:188-215).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MAX_RANK = 4  # patches.py:17


class ShapeError(ValueError):
    pass


class CoverageError(ValueError):
    pass


def grid_counts(tensor_shape, patch_shape, stride):
    """patches.py:64-70 (with validate_for, 54-62)."""
    tensor_shape = tuple(int(m) for m in tensor_shape)
    patch_shape = tuple(int(b) for b in patch_shape)
    stride = tuple(int(s) for s in stride) if stride else (1,) * len(patch_shape)
    if not 1 <= len(tensor_shape) <= MAX_RANK or any(m < 1 for m in tensor_shape):
        raise ShapeError(f"bad tensor shape {tensor_shape}")
    if len(patch_shape) != len(tensor_shape) or len(stride) != len(patch_shape):
        raise ShapeError("rank mismatch")
    if any(b < 1 for b in patch_shape) or any(s < 1 for s in stride):
        raise ShapeError("bad patch/stride")
    if any(b > m for b, m in zip(patch_shape, tensor_shape)):
        raise ShapeError("patch exceeds tensor")
    return tuple((m - b) // s + 1 for m, b, s in zip(tensor_shape, patch_shape, stride))


def _row_major_strides(shape):
    out = [1] * len(shape)
    for d in range(len(shape) - 2, -1, -1):
        out[d] = out[d + 1] * shape[d + 1]
    return np.asarray(out, dtype=np.int64)


def grid_origins(tensor_shape, patch_shape, stride):
    """Origins (N, d) int64 in row-major grid order (patches.py:107-113)."""
    counts = grid_counts(tensor_shape, patch_shape, stride)
    n = int(np.prod(counts))
    idx = np.arange(n, dtype=np.int64)
    cstr = _row_major_strides(counts)
    out = np.empty((n, len(counts)), dtype=np.int64)
    for d in range(len(counts)):
        out[:, d] = (idx // cstr[d]) % counts[d] * int(stride[d] if stride else 1)
    return out


def flat_index(tensor_shape, patch_shape, stride):
    """(N, P) flat tensor index of every (patch, offset) (patches.py:167-178)."""
    origins = grid_origins(tensor_shape, patch_shape, stride)
    tstr = _row_major_strides(tensor_shape)
    base = origins @ tstr
    offs_nd = np.indices(patch_shape).reshape(len(patch_shape), -1)
    offs = (offs_nd * tstr[:, None]).sum(axis=0)
    return base[:, None] + offs[None, :]


@dataclass
class PatchMatrix:
    values: np.ndarray
    observed: np.ndarray
    origins: np.ndarray
    means: np.ndarray
    tensor_shape: tuple
    patch_shape: tuple
    stride: tuple
    mean_subtracted: bool = False

    @property
    def num_patches(self):
        return self.values.shape[0]

    @property
    def patch_size(self):
        return self.values.shape[1]


def extract_patches(tensor, mask, patch_shape, stride=(), mean_subtract=False):
    """patches.py:125-164."""
    tensor = np.asarray(tensor, dtype=np.float64)
    patch_shape = tuple(int(b) for b in patch_shape)
    stride = tuple(int(s) for s in stride) if stride else (1,) * len(patch_shape)
    grid_counts(tensor.shape, patch_shape, stride)
    if tuple(mask.shape) != tuple(tensor.shape):
        raise ShapeError("mask shape mismatch")
    fi = flat_index(tensor.shape, patch_shape, stride)
    obs = np.asarray(mask, dtype=bool).ravel()[fi]
    vals = tensor.ravel()[fi] * obs
    n = vals.shape[0]
    means = np.zeros(n, dtype=np.float64)
    if mean_subtract:
        cnt = obs.sum(axis=1)
        ok = cnt > 0
        tot = vals.sum(axis=1)
        means[ok] = tot[ok] / cnt[ok]
        vals = (vals - means[:, None]) * obs
    return PatchMatrix(
        values=vals, observed=obs,
        origins=grid_origins(tensor.shape, patch_shape, stride),
        means=means, tensor_shape=tuple(tensor.shape),
        patch_shape=patch_shape, stride=stride, mean_subtracted=bool(mean_subtract),
    )


def coverage(tensor_shape, patch_shape, stride):
    """Analytic per-element coverage (equals patches.py:181-185's bincount)."""
    stride = tuple(stride) if stride else (1,) * len(patch_shape)
    counts = grid_counts(tensor_shape, patch_shape, stride)
    per_dim = []
    for m, b, s, g in zip(tensor_shape, patch_shape, stride, counts):
        x = np.arange(m)
        lo = np.maximum(0, -((b - 1 - x) // s))      # ceil((x-b+1)/s) clipped at 0
        hi = np.minimum(g - 1, x // s)
        per_dim.append(np.maximum(hi - lo + 1, 0))
    cov = per_dim[0]
    for c in per_dim[1:]:
        cov = np.multiply.outer(cov, c)
    return cov.astype(np.int64).reshape(tuple(tensor_shape))


def reconstitute(pm: PatchMatrix, estimates, strict=False):
    """patches.py:188-215 (sequential accumulation in ascending (i, p))."""
    est = np.asarray(estimates, dtype=np.float64)
    if est.shape != pm.values.shape:
        raise ShapeError("estimates shape mismatch")
    size = int(np.prod(pm.tensor_shape))
    fi = flat_index(pm.tensor_shape, pm.patch_shape, pm.stride).ravel()
    acc = np.zeros(size, dtype=np.float64)
    np.add.at(acc, fi, (est + pm.means[:, None]).ravel())
    cov = coverage(pm.tensor_shape, pm.patch_shape, pm.stride).ravel()
    if strict and (cov == 0).any():
        raise CoverageError(f"{int((cov == 0).sum())} elements covered by no patch")
    out = np.zeros(size, dtype=np.float64)
    np.divide(acc, cov, out=out, where=cov != 0)
    return out.reshape(pm.tensor_shape)


def apply_data_consistency(recon, original, mask, enabled=True):
    """patches.py:218-229."""
    if not enabled:
        return recon
    return np.where(np.asarray(mask, dtype=bool), original, recon)
