"""N-D patch extraction / overlap-add on the device — drop-in for
reference pkg/src/patchbeam/patches.py.

Same names, argument meaning and exceptions as the reference.  The difference
is where the data lives: a :class:`PatchMatrix` here is device-resident in the
plane-major layout (P, N); ``.values`` / ``.observed`` give (N, P) views of it
(torch CUDA tensors), ``.to_host()`` gives reference-typed numpy arrays.

Compute goes through the sm_100a kernels behind include/pb200.h
(``pb_extract_patches``, ``pb_reconstitute``, ``pb_coverage_map``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

MAX_RANK = 4  # patches.py:17


class ShapeError(ValueError):
    """Tensor / patch / mask shape mismatch (patches.py:20-21)."""


class CoverageError(ValueError):
    """Strict reconstitution found elements covered by no patch (patches.py:24-25)."""


_EXC = {_lib.PB_ESHAPE: ShapeError, _lib.PB_EVALUE: ValueError, _lib.PB_ECOVERAGE: CoverageError}


def _check_tensor_shape(shape):
    if not 1 <= len(shape) <= MAX_RANK:
        raise ShapeError(f"tensor rank must be 1..{MAX_RANK}, got {len(shape)}")
    if any(m < 1 for m in shape):
        raise ShapeError(f"tensor dims must be >= 1, got {shape}")


@dataclass(frozen=True)
class PatchSpec:
    """Patch shape and stride (patches.py:35-77)."""

    patch_shape: tuple
    stride: tuple = ()

    def __post_init__(self):
        shape = tuple(int(b) for b in self.patch_shape)
        stride = tuple(int(s) for s in self.stride) if self.stride else (1,) * len(shape)
        if len(stride) != len(shape):
            raise ShapeError("stride rank must match patch rank")
        if any(b < 1 for b in shape):
            raise ShapeError(f"patch dims must be >= 1, got {shape}")
        if any(s < 1 for s in stride):
            raise ShapeError(f"strides must be >= 1, got {stride}")
        object.__setattr__(self, "patch_shape", shape)
        object.__setattr__(self, "stride", stride)

    def validate_for(self, tensor_shape):
        _check_tensor_shape(tuple(tensor_shape))
        if len(self.patch_shape) != len(tensor_shape):
            raise ShapeError(f"patch rank {len(self.patch_shape)} != tensor rank {len(tensor_shape)}")
        for b, m in zip(self.patch_shape, tensor_shape):
            if b > m:
                raise ShapeError(f"patch shape {self.patch_shape} exceeds tensor {tuple(tensor_shape)}")

    def grid_counts(self, tensor_shape):
        self.validate_for(tuple(tensor_shape))
        return tuple((m - b) // s + 1 for m, b, s in zip(tensor_shape, self.patch_shape, self.stride))

    def num_patches(self, tensor_shape):
        return int(np.prod(self.grid_counts(tensor_shape)))

    @property
    def patch_size(self):
        return int(np.prod(self.patch_shape))

    def desc(self, tensor_shape) -> _lib.GridDesc:
        g = _lib.GridDesc()
        g.rank = len(tensor_shape)
        for d, (m, b, s) in enumerate(zip(tensor_shape, self.patch_shape, self.stride)):
            g.tensor_shape[d], g.patch_shape[d], g.stride[d] = int(m), int(b), int(s)
        return g


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def to_device(x, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (no copy if already suitable)."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if not t.is_cuda:
        t = t.cuda(non_blocking=False)
    return t.contiguous()


@dataclass
class PatchMatrix:
    """Device-resident flattened grid patches of one masked tensor (patches.py:80-104).

    values_pn (P,N) f32 — zero where unobserved, mean-subtracted if requested;
    observed_pn (P,N) uint8; means (N,) f32; counts (N,) int32 observed per patch.
    """

    values_pn: torch.Tensor
    observed_pn: torch.Tensor
    means_dev: torch.Tensor
    counts: torch.Tensor
    tensor_shape: tuple
    spec: PatchSpec
    mean_subtracted: bool = False
    n_obs: int = 0
    _cache: dict = field(default_factory=dict, repr=False)
    # code-step split of the observed-element index (pb_patch_index.split_request):
    # 0 automatic, > 0 forced threshold, < 0 never
    split_request: int = 0

    @property
    def num_patches(self):
        return self.values_pn.shape[1]

    @property
    def patch_size(self):
        return self.values_pn.shape[0]

    @property
    def values(self):
        """(N, P) view (device)."""
        return self.values_pn.T

    @property
    def observed(self):
        """(N, P) bool view (device)."""
        return self.observed_pn.view(torch.bool).T

    @property
    def means(self):
        return self.means_dev

    @property
    def origins(self):
        if "origins" not in self._cache:
            counts = self.spec.grid_counts(self.tensor_shape)
            axes = [np.arange(c, dtype=np.int64) * s for c, s in zip(counts, self.spec.stride)]
            mesh = np.meshgrid(*axes, indexing="ij")
            self._cache["origins"] = np.stack([m.ravel() for m in mesh], axis=1)
        return self._cache["origins"]

    def index(self) -> "_lib.PatchIndex":
        """Observed-element index used by the sweep (pb_build_index), built once
        per mask and refreshed if ``values``/``observed`` were edited in place
        (tracked through the tensors' version counters)."""
        c = self._cache
        ov, vv = self.observed_pn._version, self.values_pn._version
        if c.get("ix_obs_version") != ov:
            self.counts = self.observed_pn.sum(dim=0, dtype=torch.int32)
            self.n_obs = int(self.counts.sum(dtype=torch.int64).item())
            n, p = self.num_patches, self.patch_size
            nb = int(_lib.load().pb_index_bytes(n, p, self.n_obs))
            ix = _lib.PatchIndex(n, p, 0, self.n_obs, 0, None)
            ix.split_request = int(self.split_request)
            buf = torch.empty((max(nb, 1),), dtype=torch.uint8, device=self.values_pn.device)
            ix.buffer = buf.data_ptr()
            _lib.call("pb_build_index", ctypes.byref(ix), _ptr(self.observed_pn), _ptr(self.values_pn),
                      _ptr(self.counts), _stream())
            c.update(ix=ix, ix_buf=buf, ix_obs_version=ov, ix_val_version=vv)
        elif c.get("ix_val_version") != vv:
            _lib.call("pb_index_refresh_values", ctypes.byref(c["ix"]), _ptr(self.values_pn), _ptr(self.counts),
                      _stream())
            c["ix_val_version"] = vv
        return c["ix"]

    @classmethod
    def from_arrays(cls, values, observed, means=None, tensor_shape=None, spec=None):
        """Build a device PatchMatrix from reference-layout (N,P) arrays (tests /
        callers that assemble patch matrices themselves, cf. test_bpfa.py:264-293)."""
        v = np.asarray(values, dtype=np.float64)
        o = np.asarray(observed, dtype=bool)
        n, p = v.shape
        dev = torch.device("cuda")
        values_pn = torch.as_tensor(np.ascontiguousarray(np.where(o, v, 0.0).T), dtype=torch.float32, device=dev)
        obs_pn = torch.as_tensor(np.ascontiguousarray(o.T).astype(np.uint8), device=dev)
        means_t = torch.as_tensor(np.zeros(n) if means is None else np.asarray(means), dtype=torch.float32,
                                  device=dev)
        counts = obs_pn.sum(dim=0, dtype=torch.int32)
        spec = spec or PatchSpec((p,))
        return cls(values_pn, obs_pn, means_t, counts, tuple(tensor_shape or (p,)), spec, False,
                   int(o.sum()))

    def to_host(self):
        """Reference-typed numpy copy: values (N,P) f64, observed (N,P) bool, means (N,) f64."""
        return (self.values_pn.T.double().cpu().numpy(), self.observed_pn.T.bool().cpu().numpy(),
                self.means_dev.double().cpu().numpy())


def extract_patches(tensor, mask, spec: PatchSpec, mean_subtract: bool = False) -> PatchMatrix:
    """extract_patches (patches.py:125-164) on the device."""
    shape = tuple(int(m) for m in (tensor.shape))
    spec.validate_for(shape)
    if tuple(mask.shape) != shape:
        raise ShapeError(f"mask shape {tuple(mask.shape)} != tensor shape {shape}")
    if isinstance(tensor, torch.Tensor) and tensor.dtype == torch.float32:
        t = to_device(tensor)
    else:
        t = to_device(tensor, torch.float64)
    m = to_device(mask, torch.uint8) if not (isinstance(mask, torch.Tensor) and mask.dtype == torch.uint8) \
        else to_device(mask)
    if m.dtype == torch.bool:
        m = m.view(torch.uint8)
    n = spec.num_patches(shape)
    p = spec.patch_size
    dev = t.device
    values = torch.empty((p, n), dtype=torch.float32, device=dev)
    obs = torch.empty((p, n), dtype=torch.uint8, device=dev)
    means = torch.empty((n,), dtype=torch.float32, device=dev)
    counts = torch.empty((n,), dtype=torch.int32, device=dev)
    g = spec.desc(shape)
    _lib.call("pb_extract_patches", ctypes.byref(g), _ptr(t), int(t.dtype == torch.float64), _ptr(m),
              int(bool(mean_subtract)), _ptr(values), _ptr(obs), _ptr(means), _ptr(counts), _stream(),
              exc_map=_EXC)
    n_obs = int(counts.sum(dtype=torch.int64).item())
    pm = PatchMatrix(values, obs, means, counts, shape, spec, bool(mean_subtract), n_obs)
    pm._cache["mask"] = m
    return pm


def _as_estimates_pn(pm: PatchMatrix, estimates) -> torch.Tensor:
    """Accept device (N,P) views / (P,N) tensors or host (N,P) arrays -> (P,N) f32 CUDA."""
    n, p = pm.num_patches, pm.patch_size
    if isinstance(estimates, torch.Tensor):
        if tuple(estimates.shape) != (n, p):
            raise ShapeError(f"estimates shape {tuple(estimates.shape)} != patch matrix shape {(n, p)}")
        e = estimates.T
        if e.is_cuda and e.dtype == torch.float32 and e.is_contiguous():
            return e
        return to_device(e.contiguous(), torch.float32)
    est = np.asarray(estimates)
    if est.shape != (n, p):
        raise ShapeError(f"estimates shape {est.shape} != patch matrix shape {(n, p)}")
    return to_device(np.ascontiguousarray(est.T), torch.float32)


def reconstitute(pm: PatchMatrix, estimates, strict: bool = False, *, est_scale: float = 1.0,
                 dc_original=None, dc_mask=None, out: str = "host", dtype=np.float64):
    """reconstitute (patches.py:188-215): overlap-average on the device.

    Returns a numpy array of the tensor shape (``out="host"``, f64 like the
    reference) or a CUDA tensor (``out="device"``).  ``dc_original``/``dc_mask``
    fuse apply_data_consistency into the same kernel.
    """
    e = _as_estimates_pn(pm, estimates)
    io64 = dtype == np.float64 or dtype == torch.float64
    tdt = torch.float64 if io64 else torch.float32
    res = torch.empty(pm.tensor_shape, dtype=tdt, device=e.device)
    unc = torch.zeros((1,), dtype=torch.int64, device=e.device)
    dc = dc_original is not None
    orig = to_device(dc_original, tdt) if dc else None
    msk = to_device(dc_mask, torch.uint8) if dc else None
    g = pm.spec.desc(pm.tensor_shape)
    _lib.call("pb_reconstitute", ctypes.byref(g), _ptr(e), float(est_scale), _ptr(pm.means_dev), _ptr(orig),
              _ptr(msk), int(dc), int(io64), _ptr(res), _ptr(unc), _stream(), exc_map=_EXC)
    if strict:
        nu = int(unc.item())
        if nu:
            raise CoverageError(f"{nu} elements covered by no patch")
    return res.cpu().numpy() if out == "host" else res


def coverage_map(pm: PatchMatrix):
    """coverage_map (patches.py:181-185) -> numpy int array of the tensor shape."""
    res = torch.empty(pm.tensor_shape, dtype=torch.int32, device=pm.values_pn.device)
    g = pm.spec.desc(pm.tensor_shape)
    _lib.call("pb_coverage_map", ctypes.byref(g), _ptr(res), _stream(), exc_map=_EXC)
    return res.cpu().numpy().astype(np.int64)


def apply_data_consistency(recon, original, mask, enabled: bool = True):
    """apply_data_consistency (patches.py:218-229) for host arrays; the device
    path fuses it into :func:`reconstitute` (``dc_original=``, ``dc_mask=``)."""
    if tuple(recon.shape) != tuple(original.shape) or tuple(recon.shape) != tuple(mask.shape):
        raise ShapeError("data consistency requires equal shapes")
    if not enabled:
        return recon
    return np.where(np.asarray(mask, dtype=bool), original, recon)


def normalize(tensor):
    """normalize (patches.py:232-248): host pre-processing, out of the hot path."""
    tensor = np.asarray(tensor, dtype=np.float64)
    if tensor.size == 0:
        raise ShapeError("cannot normalize an empty tensor")
    if not np.isfinite(tensor).all():
        raise ValueError("tensor contains non-finite values")
    lo, hi = float(tensor.min()), float(tensor.max())
    if hi == lo:
        return np.zeros_like(tensor), 1.0, lo
    return (tensor - lo) / (hi - lo), hi - lo, lo
