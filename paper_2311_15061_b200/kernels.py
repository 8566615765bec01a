"""Drop-in for the reference's kernel module ``patchbeam._kernels``
(pkg/src/patchbeam/_kernels.py:18-145): the same seven functions with the same
names, argument order, in-place / return semantics and return types on host
numpy arrays, computed by the device seam of the C ABI (include/pb200.h:
``pb_residual_full`` ... ``pb_compose_estimates``) in f32 with f64 reductions.

The reference's bpfa calls these through the module object (bpfa.py:30), so a
maintainer can rebind them one at a time for unit-level parity::

    from patchbeam import _kernels
    from paper_2311_15061_b200 import kernels
    _kernels.code_moments = kernels.code_moments

Arrays are the reference's row-major ``(N, P)``, ``(N, K)`` and ``(K, P)`` numpy
arrays (values / weights / atoms f64, observed / usage bool); each call moves
them to the device's plane-major layouts (``(P, N)``, ``(K, N)``), runs one seam
kernel and writes back.  There is no host computation: without the library or a
GPU every call raises (``_lib.PBError`` / ``RuntimeError``).  The product path does not go
through this module: ``bpfa.gibbs_epoch`` keeps its state on the device.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .patches import _ptr, _stream


def _dev():
    if not torch.cuda.is_available():
        raise _lib.PBError(_lib.PB_ECUDA, "the kernel seam needs a CUDA device")
    return torch.device("cuda", torch.cuda.current_device())


def _pn(a, dtype=torch.float32):
    """(N, P) host array -> contiguous (P, N) device tensor."""
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).to(_dev(), dtype).contiguous()


def _u8_pn(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=bool).T).view(np.uint8)).to(_dev())


def _vec(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(_dev(), torch.float32)


def _codes(usage, weights):
    """(N, K) host codes -> (K, ld) device usage u8 / weights f32 at the library's row
    pitch (pb_code_pitch: n rounded up to 64, the aligned rows the kernels load)."""
    n, k = usage.shape
    ld = (n + 63) // 64 * 64
    z = torch.zeros((k, ld), dtype=torch.uint8, device=_dev())
    w = torch.zeros((k, ld), dtype=torch.float32, device=_dev())
    z[:, :n] = torch.from_numpy(np.ascontiguousarray(np.asarray(usage, dtype=bool).T).view(np.uint8)).to(_dev())
    w[:, :n] = torch.from_numpy(np.ascontiguousarray(np.asarray(weights, dtype=np.float64).T)).to(_dev(),
                                                                                                 torch.float32)
    return z, w, ld


def _atoms(a):
    """(K, P) host atoms -> contiguous device f32."""
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(_dev(), torch.float32)


def _check_np(resid, observed):
    if resid.shape != observed.shape or resid.ndim != 2:
        raise ValueError(f"resid {resid.shape} and observed {observed.shape} must be the same (N, P)")
    return resid.shape


def _store(out, dev_pn):
    """Write a (P, N) device result into the caller's (N, P) array in place."""
    np.copyto(out, dev_pn.T.double().cpu().numpy())


def residual_full(values, observed, usage, weights, atoms, out):
    """_kernels.py:18-31: out[i, p] = values[i, p] - sum_k usage*weights*atoms[k, p]
    on observed elements, 0 elsewhere (out written in place)."""
    n, p = _check_np(values, observed)
    k = atoms.shape[0]
    if usage.shape != (n, k) or weights.shape != (n, k) or atoms.shape != (k, p) or out.shape != (n, p):
        raise ValueError("residual_full: inconsistent shapes")
    # (device inputs held in locals until the launch: a temporary freed before it
    # would hand its memory to the next allocation)
    x, o, d = _pn(values), _u8_pn(observed), _atoms(atoms)
    z, w, ld = _codes(usage, weights)
    r = torch.empty((p, n), dtype=torch.float32, device=_dev())
    _lib.call("pb_residual_full", _ptr(x), _ptr(o), _ptr(z), _ptr(w), _ptr(d), _ptr(r), n, p, k, ld, _stream())
    _store(out, r)


def atom_moments(resid, observed, w_col):
    """_kernels.py:34-62: (A, C) with A[p] = sum_i o*w^2, C[p] = sum_i o*w*r (f64 arrays)."""
    n, p = _check_np(resid, observed)
    a = torch.empty((p,), dtype=torch.float64, device=_dev())
    c = torch.empty_like(a)
    scratch = torch.empty((2 * p * 64,), dtype=torch.float64, device=_dev())
    r, o, w = _pn(resid), _u8_pn(observed), _vec(w_col)
    _lib.call("pb_atom_moments", _ptr(r), _ptr(o), _ptr(w), n, p, _ptr(a), _ptr(c), _ptr(scratch), _stream())
    return a.cpu().numpy(), c.cpu().numpy()


def shift_atom(resid, observed, w_col, delta):
    """_kernels.py:65-74: resid[i, p] += w_col[i] * delta[p] on observed elements (in place)."""
    n, p = _check_np(resid, observed)
    r, o, w, dl = _pn(resid), _u8_pn(observed), _vec(w_col), _vec(delta)
    _lib.call("pb_shift_atom", _ptr(r), _ptr(o), _ptr(w), _ptr(dl), n, p, _stream())
    _store(resid, r)


def code_moments(resid, observed, atom):
    """_kernels.py:77-97: (u, v) with u[i] = sum_{p in Omega_i} d^2, v[i] = sum d * r (f64 arrays)."""
    n, p = _check_np(resid, observed)
    u = torch.empty((n,), dtype=torch.float32, device=_dev())
    v = torch.empty_like(u)
    r, o, d = _pn(resid), _u8_pn(observed), _vec(atom)
    _lib.call("pb_code_moments", _ptr(r), _ptr(o), _ptr(d), n, p, _ptr(u), _ptr(v), _stream())
    return u.double().cpu().numpy(), v.double().cpu().numpy()


def shift_codes(resid, observed, atom, dw):
    """_kernels.py:100-109: resid[i, p] += dw[i] * atom[p] on observed elements (in place)."""
    n, p = _check_np(resid, observed)
    r, o, d, w = _pn(resid), _u8_pn(observed), _vec(atom), _vec(dw)
    _lib.call("pb_shift_codes", _ptr(r), _ptr(o), _ptr(d), _ptr(w), n, p, _stream())
    _store(resid, r)


def masked_sq_norm(resid):
    """_kernels.py:112-130: sum of resid^2 (resid is 0 off the mask) as a Python float."""
    r = torch.from_numpy(np.ascontiguousarray(resid)).to(_dev(), torch.float32)
    out = torch.empty((1,), dtype=torch.float64, device=_dev())
    scratch = torch.empty((256,), dtype=torch.float64, device=_dev())
    _lib.call("pb_masked_sq_norm", _ptr(r), r.numel(), _ptr(out), _ptr(scratch), _stream())
    return float(out.item())


def compose_estimates(usage, weights, atoms, out):
    """_kernels.py:133-145: out[i, p] = sum_k usage*weights*atoms[k, p] (out written in place)."""
    n, k = usage.shape
    p = atoms.shape[1]
    if weights.shape != (n, k) or atoms.shape[0] != k or out.shape != (n, p):
        raise ValueError("compose_estimates: inconsistent shapes")
    est = torch.empty((p, n), dtype=torch.float32, device=_dev())
    z, w, ld = _codes(usage, weights)
    d = _atoms(atoms)
    _lib.call("pb_compose_estimates", _ptr(z), _ptr(w), _ptr(d), _ptr(est), n, p, k, ld, 0, _stream())
    _store(out, est)


__all__ = ["residual_full", "atom_moments", "shift_atom", "code_moments", "shift_codes", "masked_sq_norm",
           "compose_estimates"]
