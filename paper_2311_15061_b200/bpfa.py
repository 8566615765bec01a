"""Masked BPFA Gibbs sampling on the device — drop-in for reference
pkg/src/patchbeam/bpfa.py.

Same public names and semantics as the reference (Hyperparams, Dictionary,
GibbsState, init_state, gibbs_epoch, compose_estimates, install_dictionary,
infer, transfer_dictionary, the posterior helpers, DivergenceError).  The
sampler state is device-resident:

* ``state.dictionary.atoms`` (K,P) f32 and ``.pi`` (K,) f64 are CUDA tensors;
* ``state.usage`` / ``state.weights`` are (N,K) views (bool / f32) of the
  atom-major (K,N) device storage, so in-place edits such as the pipeline's
  warm-start ``state.usage[:] = False`` work unchanged (pipeline.py:232-233);
* ``weight_precision``, ``noise_precision`` and ``epoch`` live in a 40-byte
  device scalar block (``pb_scalars``); the first read after a sweep copies the
  block to the host once, later reads use that copy until the next sweep.

RNG modes (``rng=``):
  ``"numpy"``  — the reference's own keyed Philox4x64 streams, drawn on the
                 host and replayed on the device (rng.py:25-32, bpfa.py:293-333):
                 same seed => same draws as the reference.
  ``"philox"`` — counter-based Philox4x32-10 drawn in-kernel, π/γ drawn on the
                 device; no host round-trip per epoch (the fast path).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from .patches import PatchMatrix, PatchSpec, ShapeError, _ptr, _stream
from .rng import DOMAIN_ATOM, DOMAIN_CODE, DOMAIN_GAMMA, DOMAIN_INIT, DOMAIN_PI, keyed_rng

PRECISION_FLOOR = 1e-12  # bpfa.py:34
_PI_EPS = 1e-15          # bpfa.py:35
DEFAULT_RNG = "philox"


class DivergenceError(RuntimeError):
    """Inference produced non-finite state (bpfa.py:38-39)."""


@dataclass(frozen=True)
class Hyperparams:
    """bpfa.py:42-60."""

    num_atoms: int = 64
    concentration_a: float = 1.0
    concentration_b: float = 1.0
    weight_shape: float = 1e-6
    weight_rate: float = 1e-6
    noise_shape: float = 1e-6
    noise_rate: float = 1e-6

    def __post_init__(self):
        if self.num_atoms < 1:
            raise ValueError("num_atoms must be >= 1")
        for name in ("concentration_a", "concentration_b", "weight_shape",
                     "weight_rate", "noise_shape", "noise_rate"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be > 0")

    def as6(self):
        return (self.concentration_a, self.concentration_b, self.weight_shape,
                self.weight_rate, self.noise_shape, self.noise_rate)


@dataclass
class Dictionary:
    """K atoms (flattened patches) and activation probabilities (bpfa.py:63-80).

    ``atoms``/``pi`` may be host numpy arrays (e.g. for transfer / file I/O) or
    device tensors (inside a GibbsState)."""

    atoms: object
    pi: object
    patch_shape: tuple

    @property
    def num_atoms(self):
        return self.atoms.shape[0]

    @property
    def patch_size(self):
        return self.atoms.shape[1]

    def copy(self):
        c = (lambda a: a.clone()) if isinstance(self.atoms, torch.Tensor) else (lambda a: np.array(a, copy=True))
        return Dictionary(c(self.atoms), c(self.pi), tuple(self.patch_shape))

    def to_host(self):
        h = (lambda a: a.double().cpu().numpy()) if isinstance(self.atoms, torch.Tensor) else np.asarray
        return Dictionary(np.asarray(h(self.atoms), dtype=np.float64), np.asarray(h(self.pi), dtype=np.float64),
                          tuple(self.patch_shape))


class GibbsState:
    """Device-resident latent state of one problem (bpfa.py:83-101)."""

    def __init__(self, dictionary: Dictionary, usage_kn: torch.Tensor, weights_kn: torch.Tensor,
                 scalars: torch.Tensor, seed: int, codes_zero: bool = False):
        self.dictionary = dictionary
        self.usage_kn = usage_kn        # (K,N) uint8
        self.weights_kn = weights_kn    # (K,N) f32
        self.scalars = scalars          # 40-byte pb_scalars block (uint8 tensor)
        self.seed = int(seed)
        self._workspace = None
        self._sc_cache = None           # host copy of the scalar block (see _sc)
        self._resid_key = None          # residual in the workspace belongs to this key
        # codes known to be all zero at these tensor versions (fresh init / reset_codes)
        self._zero_key = self._codes_key() if codes_zero else None

    def _codes_key(self):
        return (self.usage_kn._version, self.weights_kn._version, id(self.usage_kn), id(self.weights_kn))

    def reset_codes(self):
        """Zero Z and S in place (the live warm start, pipeline.py:232-233) and
        remember that the next sweep may start from R = X."""
        self.usage_kn.zero_()
        self.weights_kn.zero_()
        self._zero_key = self._codes_key()

    # -- reference-shaped views -------------------------------------------
    @property
    def usage(self):
        return self.usage_kn.view(torch.bool).T

    @property
    def weights(self):
        return self.weights_kn.T

    @property
    def ld(self):
        """Row pitch of the (K, ld) code buffers."""
        return self.usage_kn.stride(0)

    @property
    def num_patches(self):
        return self.usage_kn.shape[1]

    @property
    def num_atoms(self):
        return self.usage_kn.shape[0]

    # -- device scalars ---------------------------------------------------
    def _sc(self) -> _lib.Scalars:
        """Host copy of the device scalar block.  One device->host read per change:
        the copy is kept until a sweep is launched on this state (_epoch_desc drops
        it) or the tensor is written through torch (version counter)."""
        key = (id(self.scalars), self.scalars._version)
        c = getattr(self, "_sc_cache", None)
        if c is None or c[0] != key:
            c = (key, bytes(self.scalars.cpu().numpy().tobytes()))
            self._sc_cache = c
        return _lib.Scalars.from_buffer_copy(c[1])

    def _set_sc(self, **kw):
        s = self._sc()
        for k, v in kw.items():
            setattr(s, k, v)
        self.scalars.copy_(torch.frombuffer(bytearray(bytes(s)), dtype=torch.uint8))

    weight_precision = property(lambda self: self._sc().gamma_s,
                                lambda self, v: self._set_sc(gamma_s=float(v)))
    noise_precision = property(lambda self: self._sc().gamma_eps,
                               lambda self, v: self._set_sc(gamma_eps=float(v)))
    epoch = property(lambda self: self._sc().epoch, lambda self, v: self._set_sc(epoch=int(v)))

    def to_host(self):
        """Reference-typed numpy snapshot (dict of arrays/scalars)."""
        s = self._sc()
        return dict(atoms=self.dictionary.atoms.double().cpu().numpy(),
                    pi=self.dictionary.pi.double().cpu().numpy(),
                    usage=self.usage_kn.T.bool().cpu().numpy(),
                    weights=self.weights_kn.T.double().cpu().numpy(),
                    weight_precision=s.gamma_s, noise_precision=s.gamma_eps, epoch=s.epoch, seed=self.seed)

    @classmethod
    def from_host(cls, atoms, pi, usage, weights, weight_precision, noise_precision, epoch, seed,
                  patch_shape=(), device="cuda"):
        """Upload a reference-typed state ((N,K) usage/weights, (K,P) atoms)."""
        atoms_t = torch.as_tensor(np.asarray(atoms, dtype=np.float32), device=device).contiguous()
        pi_t = torch.as_tensor(np.asarray(pi, dtype=np.float64), device=device).contiguous()
        k, n = np.asarray(atoms).shape[0], np.asarray(usage).shape[0]
        u, w = _alloc_codes(k, n, torch.device(device))
        u.copy_(torch.as_tensor(np.ascontiguousarray(np.asarray(usage, dtype=np.uint8).T)))
        w.copy_(torch.as_tensor(np.ascontiguousarray(np.asarray(weights, dtype=np.float32).T)))
        sc = _make_scalars(weight_precision, noise_precision, epoch, device)
        return cls(Dictionary(atoms_t, pi_t, tuple(patch_shape)), u, w, sc, seed)

    def workspace(self, n, p, k, nnz):
        key = (n, p, k, nnz)
        if self._workspace is None or self._workspace[0] != key:
            nb = int(_lib.load().pb_epoch_workspace_bytes(n, p, k, nnz))
            self._workspace = (key, torch.empty((nb,), dtype=torch.uint8, device=self.usage_kn.device),
                               torch.empty((k,), dtype=torch.int32, device=self.usage_kn.device))
        return self._workspace[1], self._workspace[2]


def _alloc_codes(k, n, device):
    """Zeroed (K, N) usage/weights views of row-pitched (K, ld) buffers
    (ld = pb_code_pitch(N): aligned vector loads in the dictionary step)."""
    ld = int(_lib.load().pb_code_pitch(n))
    u = torch.zeros((k, ld), dtype=torch.uint8, device=device)
    w = torch.zeros((k, ld), dtype=torch.float32, device=device)
    return u[:, :n], w[:, :n]


def _make_scalars(gs, ge, epoch, device):
    s = _lib.Scalars(float(gs), float(ge), 0.0, 0.0, int(epoch), 0)
    return torch.frombuffer(bytearray(bytes(s)), dtype=torch.uint8).to(device)


def _prior_atoms(seed, k, p_len):
    """bpfa.py:121-122 — drawn from the reference's exact stream (seed, 1)."""
    return keyed_rng(seed, DOMAIN_INIT).standard_normal((k, p_len)) / math.sqrt(p_len)


def init_state(pm: PatchMatrix, hp: Hyperparams, seed: int, init_mode: str = "data") -> GibbsState:
    """bpfa.py:104-152.  Data mode seeds atoms from the K patches with the most
    observed elements (ties by index), unit-normalized; surplus atoms keep prior draws."""
    n, p_len = pm.num_patches, pm.patch_size
    if n < 1 or p_len < 1:
        raise ShapeError("patch matrix must be non-empty")
    k = hp.num_atoms
    atoms = _prior_atoms(seed, k, p_len)
    if init_mode == "data":
        counts = pm.counts.cpu().numpy()
        order = np.argsort(-counts, kind="stable")
        take = min(k, n)
        idx = torch.as_tensor(order[:take], device=pm.values_pn.device)
        cand = pm.values_pn.index_select(1, idx).T.double().cpu().numpy()
        norms = np.sqrt((cand * cand).sum(axis=1))
        ok = norms > 0
        atoms = atoms.copy()
        atoms[:take][ok] = cand[ok] / norms[ok, None]
    elif init_mode != "prior":
        raise ValueError(f"unknown init mode {init_mode!r}")
    dev = pm.values_pn.device
    pi0 = hp.concentration_a / (hp.concentration_a + hp.concentration_b)
    d = Dictionary(torch.as_tensor(atoms, dtype=torch.float32, device=dev).contiguous(),
                   torch.full((k,), pi0, dtype=torch.float64, device=dev), tuple(pm.spec.patch_shape))
    return GibbsState(d, *_alloc_codes(k, n, dev),
                      _make_scalars(max(hp.weight_shape / hp.weight_rate, PRECISION_FLOOR),
                                    max(hp.noise_shape / hp.noise_rate, PRECISION_FLOOR), 0, dev), seed,
                      codes_zero=True)


def install_dictionary(state_seed: int, pm: PatchMatrix, hp: Hyperparams, dictionary: Dictionary) -> GibbsState:
    """bpfa.py:355-376."""
    if dictionary.patch_size != pm.patch_size:
        raise ShapeError(f"dictionary patch size {dictionary.patch_size} != patches {pm.patch_size}")
    n, k, dev = pm.num_patches, dictionary.num_atoms, pm.values_pn.device
    atoms = torch.as_tensor(np.asarray(dictionary.atoms.cpu() if isinstance(dictionary.atoms, torch.Tensor)
                                       else dictionary.atoms), dtype=torch.float32, device=dev).contiguous()
    pi = torch.as_tensor(np.asarray(dictionary.pi.cpu() if isinstance(dictionary.pi, torch.Tensor)
                                    else dictionary.pi), dtype=torch.float64, device=dev).contiguous()
    return GibbsState(Dictionary(atoms, pi, tuple(dictionary.patch_shape)),
                      *_alloc_codes(k, n, dev),
                      _make_scalars(max(hp.weight_shape / hp.weight_rate, PRECISION_FLOOR),
                                    max(hp.noise_shape / hp.noise_rate, PRECISION_FLOOR), 0, dev), state_seed,
                      codes_zero=True)


# --- the sweep ---------------------------------------------------------------

def _resid_key(state: GibbsState, pm: PatchMatrix, ws):
    a = state.dictionary.atoms
    return (id(pm), pm.values_pn._version, pm.observed_pn._version, id(pm._cache.get("ix_buf")),
            state._codes_key(), id(a), a._version, ws.data_ptr())


def _epoch_desc(state: GibbsState, pm: PatchMatrix, hp: Hyperparams, freeze: bool, mode: int):
    n, p, k = pm.num_patches, pm.patch_size, state.num_atoms
    ix = pm.index()
    ws, m = state.workspace(n, p, k, pm.n_obs)
    d = _lib.EpochDesc()
    key = _resid_key(state, pm, ws)
    if state._resid_key == key:
        d.resid_mode = _lib.PB_RESID_CARRY            # residual of this exact state is resident
    elif state._zero_key == state._codes_key():
        d.resid_mode = _lib.PB_RESID_FROM_VALUES      # Z*S == 0  =>  R = X
        d.codes_zero = 1                              # Z = S = 0: the code step reads no old state
    else:
        d.resid_mode = _lib.PB_RESID_RECOMPUTE        # residual_full (bpfa.py:297)
    state._resid_key = key
    d.index = ctypes.pointer(ix)
    d.counts = pm.counts.data_ptr()
    d.n, d.p, d.k = n, p, k
    d.ld = state.ld
    d.freeze_dict = int(bool(freeze))
    d.rng_mode = mode
    d.seed = state.seed & 0xFFFFFFFFFFFFFFFF
    d.n_obs = pm.n_obs
    for j, v in enumerate(_hyper6(hp)):
        d.hyper[j] = float(v)
    d.values, d.observed = pm.values_pn.data_ptr(), pm.observed_pn.data_ptr()
    d.atoms, d.pi = state.dictionary.atoms.data_ptr(), state.dictionary.pi.data_ptr()
    d.usage, d.weights = state.usage_kn.data_ptr(), state.weights_kn.data_ptr()
    d.scalars = state.scalars.data_ptr()
    state._sc_cache = None   # the sweep rewrites the scalar block on the device
    d.workspace = ws.data_ptr()
    return d, m


def _hyper6(hp):
    """(a, b, c, d, e, f) of a Hyperparams — this package's or the reference's
    dataclass (bpfa.py:42-60), so reference callers can pass theirs."""
    return (hp.concentration_a, hp.concentration_b, hp.weight_shape, hp.weight_rate, hp.noise_shape, hp.noise_rate)


def _check_state(state, pm):
    if state.num_patches != pm.num_patches or state.dictionary.patch_size != pm.patch_size:
        raise ShapeError("state dimensions do not match the patch matrix")
    a = state.dictionary.atoms
    if a.dtype != torch.float32 or not a.is_contiguous():
        state.dictionary.atoms = a.to(torch.float32).contiguous()
    if state.dictionary.pi.dtype != torch.float64 or not state.dictionary.pi.is_contiguous():
        state.dictionary.pi = state.dictionary.pi.to(torch.float64).contiguous()


def reference_draws(seed, epoch, k_len, n, p_len, freeze):
    """The reference's exact per-epoch draws (bpfa.py:304, 310, 258-259), (K,·) f64."""
    atom = None
    if not freeze:
        atom = np.stack([keyed_rng(seed, DOMAIN_ATOM, epoch, k).standard_normal(p_len) for k in range(k_len)])
    cu = np.empty((k_len, n))
    cg = np.empty((k_len, n))
    for k in range(k_len):
        r = keyed_rng(seed, DOMAIN_CODE, epoch, k)
        cu[k] = r.random(n)
        cg[k] = r.standard_normal(n)
    return atom, cu, cg


def gibbs_epoch(state: GibbsState, pm: PatchMatrix, hp: Hyperparams, freeze_dict: bool = False,
                rng: str | None = None, draws=None, check: bool = True) -> GibbsState:
    """One full sweep (bpfa.py:278-345); mutates and returns ``state`` with epoch + 1.

    ``draws`` (numpy mode only) may supply (atom (K,P), code_u (K,N), code_g (K,N))
    for this epoch; by default they are drawn from the reference streams."""
    rng = rng or DEFAULT_RNG
    _check_state(state, pm)
    n, p, k = pm.num_patches, pm.patch_size, state.num_atoms
    if rng == "philox":
        d, m = _epoch_desc(state, pm, hp, freeze_dict, _lib.PB_RNG_PHILOX)
        _lib.call("pb_gibbs_epoch", ctypes.byref(d), _ptr(m), _stream())
        if check:
            s = state._sc()
            if s.diverged:
                raise DivergenceError(f"non-finite state at epoch {s.epoch}: gamma_s={s.gamma_s}, "
                                      f"gamma_eps={s.gamma_eps}, masked residual norm={s.sq_r}")
        return state
    if rng != "numpy":
        raise ValueError(f"unknown rng mode {rng!r}")
    epoch = state.epoch + 1
    atom, cu, cg = draws if draws is not None else reference_draws(state.seed, epoch, k, n, p, freeze_dict)
    dev = state.usage_kn.device
    t_atom = torch.as_tensor(np.ascontiguousarray(atom, dtype=np.float64), device=dev) if atom is not None else None
    t_u = torch.as_tensor(np.ascontiguousarray(cu, dtype=np.float64), device=dev)
    t_g = torch.as_tensor(np.ascontiguousarray(cg, dtype=np.float64), device=dev)
    d, m = _epoch_desc(state, pm, hp, freeze_dict, _lib.PB_RNG_REPLAY)
    d.atom_draws = t_atom.data_ptr() if t_atom is not None else None
    d.code_u, d.code_g = t_u.data_ptr(), t_g.data_ptr()
    _lib.call("pb_gibbs_epoch", ctypes.byref(d), _ptr(m), _stream())
    # pi / gamma draws from the reference streams (bpfa.py:313-333)
    mk = m.cpu().numpy().astype(np.float64)
    s = state._sc()
    sh_a = hp.concentration_a / k + mk
    sh_b = hp.concentration_b * (k - 1) / k + n - mk
    pi = keyed_rng(state.seed, DOMAIN_PI, epoch).beta(np.maximum(sh_a, PRECISION_FLOOR),
                                                       np.maximum(sh_b, PRECISION_FLOOR))
    g5 = keyed_rng(state.seed, DOMAIN_GAMMA, epoch)
    gs = max(g5.gamma(hp.weight_shape + 0.5 * n * k, 1.0 / (hp.weight_rate + 0.5 * s.sq_w)), PRECISION_FLOOR)
    ge = max(g5.gamma(hp.noise_shape + 0.5 * pm.n_obs, 1.0 / (hp.noise_rate + 0.5 * s.sq_r)), PRECISION_FLOOR)
    state.dictionary.pi.copy_(torch.as_tensor(pi, dtype=torch.float64))
    s.gamma_s, s.gamma_eps, s.epoch = gs, ge, epoch
    state.scalars.copy_(torch.frombuffer(bytearray(bytes(s)), dtype=torch.uint8))
    if not (math.isfinite(gs) and math.isfinite(ge) and math.isfinite(s.sq_r)):
        raise DivergenceError(f"non-finite state at epoch {epoch}: gamma_s={gs}, gamma_eps={ge}, "
                              f"masked residual norm={s.sq_r}")
    return state


def compose_estimates(state: GibbsState, out: torch.Tensor | None = None, accumulate: bool = False):
    """bpfa.py:348-352 -> (N,P) device view of a (P,N) f32 tensor."""
    k, n = state.usage_kn.shape
    p = state.dictionary.patch_size
    if out is None:
        out = torch.empty((p, n), dtype=torch.float32, device=state.usage_kn.device)
    _lib.call("pb_compose_estimates", _ptr(state.usage_kn), _ptr(state.weights_kn),
              _ptr(state.dictionary.atoms), _ptr(out), n, p, k, state.ld, int(accumulate), _stream())
    return out.T


def infer(pm: PatchMatrix, hp: Hyperparams, epochs: int, seed: int, freeze_dict: bool = False,
          initial_dict: Dictionary | None = None, init_mode: str = "data", average_last: int = 1,
          state: GibbsState | None = None, rng: str | None = None):
    """bpfa.py:379-414: run `epochs` sweeps; returns (state, estimates (N,P) device view)."""
    if epochs < 1:
        raise ValueError("epochs must be >= 1")
    rng = rng or DEFAULT_RNG
    if state is None:
        if initial_dict is not None:
            if hp.num_atoms != initial_dict.num_atoms:
                hp = replace(hp, num_atoms=initial_dict.num_atoms)
            state = install_dictionary(seed, pm, hp, initial_dict)
        elif not freeze_dict and init_mode == "data":
            # bpfa.py:126-134 data-init atoms are overwritten before first use
            # when the dictionary step runs (Z=0 => lambda=P, mu=0; SURVEY App. A
            # Q1), so the top-K gather can be skipped with identical results.
            state = init_state(pm, hp, seed, init_mode="prior")
        else:
            state = init_state(pm, hp, seed, init_mode=init_mode)
    average_last = max(1, min(int(average_last), epochs))
    tail = None
    for t in range(epochs):
        gibbs_epoch(state, pm, hp, freeze_dict=freeze_dict, rng=rng, check=(rng == "numpy" or t == epochs - 1))
        if t >= epochs - average_last:
            e = compose_estimates(state, out=tail, accumulate=tail is not None)
            tail = e.T
    est = tail.T
    if average_last > 1:
        est = (tail / average_last).T
    return state, est


def transfer_dictionary(src: Dictionary, dst_patch_shape, dst_tensor_shape=None) -> Dictionary:
    """bpfa.py:417-458: re-shape a dictionary for a destination problem.

    Equal patch shapes copy the atoms bitwise; a destination patch shape that
    extends the source's with extra trailing dimensions (which must span the
    destination tensor) re-uses each source atom across every slice of them,
    tiled and renormalized — on the device (pb_transfer_atoms).  Host atoms give
    a host (f64) dictionary, device atoms a device (f32) one."""
    dst = tuple(int(b) for b in dst_patch_shape)
    sshape = tuple(src.patch_shape)
    ds, dd = len(sshape), len(dst)
    repeat, normalize = 1, 0
    if dst != sshape:
        if dd <= ds or dst[:ds] != sshape:
            raise ShapeError(f"cannot transfer atoms of shape {sshape} to patch shape {dst}")
        extra = dst[ds:]
        if dst_tensor_shape is not None:
            if len(dst_tensor_shape) != dd:
                raise ShapeError("destination tensor rank does not match its patch shape")
            for i, b in enumerate(extra, start=ds):
                if b != dst_tensor_shape[i]:
                    raise ShapeError(f"transfer dimension {i} must span the destination tensor "
                                     f"({b} != {dst_tensor_shape[i]})")
        repeat, normalize = int(np.prod(extra)), 1
    on_dev = isinstance(src.atoms, torch.Tensor)
    if not normalize:
        return src.copy()
    a = src.atoms if on_dev else torch.as_tensor(np.asarray(src.atoms, dtype=np.float32))
    a = a.to(device="cuda", dtype=torch.float32).contiguous()
    k, sp = a.shape
    out = torch.empty((k, sp * repeat), dtype=torch.float32, device=a.device)
    _lib.call("pb_transfer_atoms", _ptr(a), k, sp, repeat, normalize, _ptr(out), _stream())
    if on_dev:
        pi = src.pi.clone() if isinstance(src.pi, torch.Tensor) else torch.as_tensor(np.asarray(src.pi), device="cuda")
        return Dictionary(out, pi, dst)
    return Dictionary(out.double().cpu().numpy(), np.array(src.pi, dtype=np.float64, copy=True), dst)


# --- posterior helpers (bpfa.py:189-235), via the fine-grained seam kernels ----

def _residual(pm: PatchMatrix, state: GibbsState) -> torch.Tensor:
    """bpfa.py:181-186 -> (P,N) f32 device."""
    out = torch.empty_like(pm.values_pn)
    _lib.call("pb_residual_full", _ptr(pm.values_pn), _ptr(pm.observed_pn), _ptr(state.usage_kn),
              _ptr(state.weights_kn), _ptr(state.dictionary.atoms), _ptr(out), pm.num_patches, pm.patch_size,
              state.num_atoms, state.ld, _stream())
    return out


def _w_col(state, k):
    return torch.where(state.usage_kn[k].bool(), state.weights_kn[k], torch.zeros((), device=state.weights_kn.device))


def atom_posterior(pm: PatchMatrix, state: GibbsState, k: int):
    """Per-pixel (lambda, mu) of atom k (bpfa.py:189-196) -> numpy f64."""
    r = _residual(pm, state)
    dev = r.device
    a = torch.empty((pm.patch_size,), dtype=torch.float64, device=dev)
    c = torch.empty_like(a)
    scratch = torch.empty((2 * pm.patch_size * 64,), dtype=torch.float64, device=dev)
    w = _w_col(state, k).contiguous()
    _lib.call("pb_atom_moments", _ptr(r), _ptr(pm.observed_pn), _ptr(w), pm.num_patches, pm.patch_size,
              _ptr(a), _ptr(c), _ptr(scratch), _stream())
    a, c = a.cpu().numpy(), c.cpu().numpy()
    ge = state.noise_precision
    atom = state.dictionary.atoms[k].double().cpu().numpy()
    lam = pm.patch_size + ge * a
    return lam, ge * (c + atom * a) / lam


def code_posterior(pm: PatchMatrix, state: GibbsState, k: int):
    """Per-patch (log_rho, alpha, mean) of atom k (bpfa.py:199-214) -> numpy f64."""
    r = _residual(pm, state)
    n = pm.num_patches
    u = torch.empty((n,), dtype=torch.float32, device=r.device)
    v = torch.empty_like(u)
    atom = state.dictionary.atoms[k].contiguous()
    _lib.call("pb_code_moments", _ptr(r), _ptr(pm.observed_pn), _ptr(atom), n, pm.patch_size, _ptr(u), _ptr(v),
              _stream())
    u, v = u.double().cpu().numpy(), v.double().cpu().numpy()
    s_old = state.weights_kn[k].double().cpu().numpy()
    w_old = np.where(state.usage_kn[k].cpu().numpy() != 0, s_old, 0.0)
    gs, ge = state.weight_precision, state.noise_precision
    proj = v + w_old * u
    pk = float(np.clip(float(state.dictionary.pi[k]), _PI_EPS, 1.0 - _PI_EPS))
    log_rho = (math.log(pk) - math.log1p(-pk)) - 0.5 * ge * (s_old * s_old * u - 2.0 * s_old * proj)
    alpha = gs + ge * u
    return log_rho, alpha, ge * proj / alpha


def pi_posterior(state: GibbsState, hp: Hyperparams):
    """bpfa.py:217-222."""
    n, k = state.num_patches, state.num_atoms
    m = state.usage_kn.sum(dim=1, dtype=torch.int64).double().cpu().numpy()
    return hp.concentration_a / k + m, hp.concentration_b * (k - 1) / k + n - m


def gamma_posteriors(pm: PatchMatrix, state: GibbsState, hp: Hyperparams):
    """bpfa.py:225-235."""
    n, k = state.num_patches, state.num_atoms
    dev = pm.values_pn.device
    scratch = torch.empty((256,), dtype=torch.float64, device=dev)
    out = torch.empty((1,), dtype=torch.float64, device=dev)
    _lib.call("pb_masked_sq_norm", _ptr(state.weights_kn), state.ld * k, _ptr(out), _ptr(scratch), _stream())
    sq_w = float(out.item())
    r = _residual(pm, state)
    _lib.call("pb_masked_sq_norm", _ptr(r), n * pm.patch_size, _ptr(out), _ptr(scratch), _stream())
    sq_r = float(out.item())
    return ((hp.weight_shape + 0.5 * n * k, hp.weight_rate + 0.5 * sq_w),
            (hp.noise_shape + 0.5 * pm.n_obs, hp.noise_rate + 0.5 * sq_r))
