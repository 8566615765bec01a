"""ORACLE (test infrastructure only): ctypes binding of oracle/csrc/oracle_kernels.c.

The C file restates reference pkg/src/patchbeam/_kernels.py:18-145 with the
same loop and reduction order.  Built by ``oracle/Makefile`` (``build()`` in
__graft_entry__ runs it); built on first use if absent.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or (
        os.path.getmtime(_SO) < os.path.getmtime(os.path.join(_HERE, "csrc", "oracle_kernels.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_SO)
            P = ctypes.c_void_p
            I = ctypes.c_int64
            L.oracle_residual_full.argtypes = [P, P, P, P, P, P, I, I, I]
            L.oracle_atom_moments.argtypes = [P, P, P, P, P, I, I]
            L.oracle_shift_atom.argtypes = [P, P, P, P, I, I]
            L.oracle_code_moments.argtypes = [P, P, P, P, P, I, I]
            L.oracle_shift_codes.argtypes = [P, P, P, P, I, I]
            L.oracle_masked_sq_norm.argtypes = [P, I, I]
            L.oracle_masked_sq_norm.restype = ctypes.c_double
            L.oracle_compose_estimates.argtypes = [P, P, P, P, I, I, I]
            L.oracle_num_threads.restype = ctypes.c_int
            for fn in ("oracle_residual_full", "oracle_atom_moments", "oracle_shift_atom",
                       "oracle_code_moments", "oracle_shift_codes", "oracle_compose_estimates"):
                getattr(L, fn).restype = None
            _lib = L
    return _lib


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _u8(a):
    return np.ascontiguousarray(a).view(np.uint8) if a.dtype == np.bool_ else np.ascontiguousarray(a, dtype=np.uint8)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def residual_full(values, observed, usage, weights, atoms, out):
    n, p = values.shape
    k = atoms.shape[0]
    v, o, z, w, d = _f64(values), _u8(observed), _u8(usage), _f64(weights), _f64(atoms)
    assert out.flags.c_contiguous and out.dtype == np.float64
    lib().oracle_residual_full(_p(v), _p(o), _p(z), _p(w), _p(d), _p(out), n, p, k)


def atom_moments(resid, observed, w_col):
    n, p = resid.shape
    a = np.empty(p)
    c = np.empty(p)
    r, o, w = _f64(resid), _u8(observed), _f64(w_col)
    lib().oracle_atom_moments(_p(r), _p(o), _p(w), _p(a), _p(c), n, p)
    return a, c


def shift_atom(resid, observed, w_col, delta):
    n, p = resid.shape
    assert resid.flags.c_contiguous and resid.dtype == np.float64
    o, w, dl = _u8(observed), _f64(w_col), _f64(delta)
    lib().oracle_shift_atom(_p(resid), _p(o), _p(w), _p(dl), n, p)


def code_moments(resid, observed, atom):
    n, p = resid.shape
    u = np.empty(n)
    v = np.empty(n)
    r, o, d = _f64(resid), _u8(observed), _f64(atom)
    lib().oracle_code_moments(_p(r), _p(o), _p(d), _p(u), _p(v), n, p)
    return u, v


def shift_codes(resid, observed, atom, dw):
    n, p = resid.shape
    assert resid.flags.c_contiguous and resid.dtype == np.float64
    o, d, w = _u8(observed), _f64(atom), _f64(dw)
    lib().oracle_shift_codes(_p(resid), _p(o), _p(d), _p(w), n, p)


def masked_sq_norm(resid):
    n, p = resid.shape
    r = _f64(resid)
    return float(lib().oracle_masked_sq_norm(_p(r), n, p))


def compose_estimates(usage, weights, atoms, out):
    n, k = usage.shape
    p = atoms.shape[1]
    z, w, d = _u8(usage), _f64(weights), _f64(atoms)
    lib().oracle_compose_estimates(_p(z), _p(w), _p(d), _p(out), n, k, p)


def num_threads() -> int:
    return int(lib().oracle_num_threads())
