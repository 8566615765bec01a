"""ORACLE (test infrastructure only): masked BPFA Gibbs sampler, f64.

Restates reference pkg/src/patchbeam/bpfa.py.  Heavy loops go through the C
restatement of the reference's Numba kernels (oracle/_ckernels.py); the
elementwise conditional algebra is the same numpy expressions evaluated in the
same order, so a run is bit-identical to the reference for the same seed
(pinned by tests/test_oracle_golden.py against tests/golden/*.npz).

Draw schedule (reference bpfa.py:293-333, rng.py):
  init                (seed, 1)            standard_normal((K, P))
  atom k, epoch e     (seed, 2, e, k)      standard_normal(P)
  codes k, epoch e    (seed, 3, e, k)      random(N) then standard_normal(N)
  pi, epoch e         (seed, 4, e)         beta(a_vec, b_vec)
  gammas, epoch e     (seed, 5, e)         gamma(gamma_s) then gamma(gamma_eps)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _ckernels as ck
from .rng import DOMAIN_ATOM, DOMAIN_CODE, DOMAIN_GAMMA, DOMAIN_INIT, DOMAIN_PI, keyed_rng

FLOOR = 1e-12      # bpfa.py:34
PI_EPS = 1e-15     # bpfa.py:35


class DivergenceError(RuntimeError):
    pass


@dataclass
class Hyper:
    """bpfa.py:42-60 (field names match the reference Hyperparams)."""
    num_atoms: int = 64
    concentration_a: float = 1.0
    concentration_b: float = 1.0
    weight_shape: float = 1e-6
    weight_rate: float = 1e-6
    noise_shape: float = 1e-6
    noise_rate: float = 1e-6


@dataclass
class State:
    """bpfa.py:63-101 flattened: atoms (K,P), pi (K,), usage (N,K) bool, weights (N,K)."""
    atoms: np.ndarray
    pi: np.ndarray
    usage: np.ndarray
    weights: np.ndarray
    gamma_s: float
    gamma_eps: float
    epoch: int
    seed: int

    def copy(self):
        return State(self.atoms.copy(), self.pi.copy(), self.usage.copy(), self.weights.copy(),
                     float(self.gamma_s), float(self.gamma_eps), int(self.epoch), int(self.seed))


class StreamDraws:
    """Draws from the reference's keyed streams; optionally records them."""

    def __init__(self, seed: int, record: bool = False):
        self.seed = int(seed)
        self.record = record
        self.log: dict = {}

    def atom(self, epoch, k, p_len):
        g = keyed_rng(self.seed, DOMAIN_ATOM, epoch, k).standard_normal(p_len)
        if self.record:
            self.log[("atom", epoch, k)] = g
        return g

    def codes(self, epoch, k, n):
        r = keyed_rng(self.seed, DOMAIN_CODE, epoch, k)
        u = r.random(n)
        g = r.standard_normal(n)
        if self.record:
            self.log[("code", epoch, k)] = (u, g)
        return u, g

    def pi_rng(self, epoch):
        return keyed_rng(self.seed, DOMAIN_PI, epoch)

    def gamma_rng(self, epoch):
        return keyed_rng(self.seed, DOMAIN_GAMMA, epoch)


def prior_atoms(seed, k, p_len):
    """bpfa.py:121-122."""
    return keyed_rng(seed, DOMAIN_INIT).standard_normal((k, p_len)) / math.sqrt(p_len)


def init_state(pm, hp, seed, init_mode="data") -> State:
    """bpfa.py:104-152."""
    n, p_len = pm.values.shape
    k = int(hp.num_atoms)
    atoms = prior_atoms(seed, k, p_len)
    if init_mode == "data":
        atoms = atoms.copy()
        order = np.argsort(-pm.observed.sum(axis=1), kind="stable")
        m = min(k, n)
        cand = pm.values[order[:m]].astype(np.float64)
        nrm = np.sqrt((cand * cand).sum(axis=1))
        good = nrm > 0
        atoms[:m][good] = cand[good] / nrm[good, None]
    elif init_mode != "prior":
        raise ValueError(init_mode)
    pi0 = hp.concentration_a / (hp.concentration_a + hp.concentration_b)
    return State(
        atoms=atoms, pi=np.full(k, pi0, dtype=np.float64),
        usage=np.zeros((n, k), dtype=bool), weights=np.zeros((n, k), dtype=np.float64),
        gamma_s=max(hp.weight_shape / hp.weight_rate, FLOOR),
        gamma_eps=max(hp.noise_shape / hp.noise_rate, FLOOR),
        epoch=0, seed=int(seed),
    )


def install_dictionary(seed, pm, hp, atoms, pi) -> State:
    """bpfa.py:355-376."""
    n = pm.values.shape[0]
    k = atoms.shape[0]
    return State(
        atoms=np.array(atoms, dtype=np.float64), pi=np.array(pi, dtype=np.float64),
        usage=np.zeros((n, k), dtype=bool), weights=np.zeros((n, k), dtype=np.float64),
        gamma_s=max(hp.weight_shape / hp.weight_rate, FLOOR),
        gamma_eps=max(hp.noise_shape / hp.noise_rate, FLOOR),
        epoch=0, seed=int(seed),
    )


# --- conditional algebra (bpfa.py:161-178) ---------------------------------

def atom_params(mom_a, mom_c, atom, g_eps, p_len):
    with np.errstate(invalid="ignore", over="ignore"):
        lam = p_len + g_eps * mom_a
        mu = g_eps * (mom_c + atom * mom_a) / lam
    return lam, mu


def code_params(u, v, w_old, s_old, pi_k, g_s, g_eps):
    with np.errstate(invalid="ignore", over="ignore"):
        proj = v + w_old * u
        pk = np.clip(pi_k, PI_EPS, 1.0 - PI_EPS)
        lo = np.log(pk) - np.log1p(-pk)
        log_rho = lo - 0.5 * g_eps * (s_old * s_old * u - 2.0 * s_old * proj)
        alpha = g_s + g_eps * u
        mean = g_eps * proj / alpha
    return log_rho, alpha, mean


def residual(pm, st):
    """bpfa.py:181-186."""
    out = np.empty_like(pm.values, dtype=np.float64)
    ck.residual_full(pm.values, pm.observed, st.usage, st.weights, st.atoms, out)
    return out


def active_weights(st, k):
    return np.where(st.usage[:, k], st.weights[:, k], 0.0)


def atom_posterior(pm, st, k):
    """bpfa.py:189-196."""
    r = residual(pm, st)
    a, c = ck.atom_moments(r, pm.observed, active_weights(st, k))
    return atom_params(a, c, st.atoms[k], st.gamma_eps, float(pm.values.shape[1]))


def code_posterior(pm, st, k):
    """bpfa.py:199-214."""
    r = residual(pm, st)
    u, v = ck.code_moments(r, pm.observed, st.atoms[k])
    s_old = st.weights[:, k]
    return code_params(u, v, active_weights(st, k), s_old, float(st.pi[k]), st.gamma_s, st.gamma_eps)


def pi_posterior(st, hp):
    """bpfa.py:217-222."""
    n, k = st.usage.shape
    m = st.usage.sum(axis=0).astype(np.float64)
    return hp.concentration_a / k + m, hp.concentration_b * (k - 1) / k + n - m


def gamma_posteriors(pm, st, hp):
    """bpfa.py:225-235."""
    n, k = st.usage.shape
    sw = float((st.weights * st.weights).sum())
    r = residual(pm, st)
    n_obs = int(pm.observed.sum())
    sr = ck.masked_sq_norm(r)
    return (hp.weight_shape + 0.5 * n * k, hp.weight_rate + 0.5 * sw), \
           (hp.noise_shape + 0.5 * n_obs, hp.noise_rate + 0.5 * sr)


# --- the sweep (bpfa.py:240-345) ---------------------------------------------

def sample_codes(resid, pm, st, k, u_draw, g_draw):
    """bpfa.py:240-275 with the (uniform, normal) draws supplied."""
    d = st.atoms[k]
    u, v = ck.code_moments(resid, pm.observed, d)
    s_old = st.weights[:, k].copy()
    w_old = np.where(st.usage[:, k], s_old, 0.0)
    log_rho, alpha, mean = code_params(u, v, w_old, s_old, float(st.pi[k]), st.gamma_s, st.gamma_eps)
    z = (np.log(u_draw) - np.log1p(-u_draw)) < log_rho
    s_new = np.where(z, mean + g_draw / np.sqrt(alpha), g_draw / math.sqrt(st.gamma_s))
    w_new = np.where(z, s_new, 0.0)
    ck.shift_codes(resid, pm.observed, d, w_old - w_new)
    st.usage[:, k] = z
    st.weights[:, k] = s_new


def gibbs_epoch(st: State, pm, hp, freeze_dict=False, draws=None, trace=None) -> State:
    """bpfa.py:278-345.  Mutates and returns ``st``.

    ``trace`` (dict) optionally receives intermediate quantities for
    teacher-forced checks: the atoms after the dictionary step, m_k, sums.
    """
    n, p_len = pm.values.shape
    if st.usage.shape[0] != n or st.atoms.shape[1] != p_len:
        raise ValueError("state dimensions do not match the patch matrix")
    k_len = st.atoms.shape[0]
    epoch = st.epoch + 1
    draws = draws if draws is not None else StreamDraws(st.seed)

    r = residual(pm, st)
    if not freeze_dict:
        for k in range(k_len):
            w = active_weights(st, k)
            a, c = ck.atom_moments(r, pm.observed, w)
            lam, mu = atom_params(a, c, st.atoms[k], st.gamma_eps, float(p_len))
            new = mu + draws.atom(epoch, k, p_len) / np.sqrt(lam)
            ck.shift_atom(r, pm.observed, w, st.atoms[k] - new)
            st.atoms[k] = new
    if trace is not None:
        trace["atoms_after_dict"] = st.atoms.copy()
    for k in range(k_len):
        ud, gd = draws.codes(epoch, k, n)
        sample_codes(r, pm, st, k, ud, gd)

    sh_a, sh_b = pi_posterior(st, hp)
    st.pi = draws.pi_rng(epoch).beta(np.maximum(sh_a, FLOOR), np.maximum(sh_b, FLOOR))

    g5 = draws.gamma_rng(epoch)
    sw = float((st.weights * st.weights).sum())
    st.gamma_s = max(g5.gamma(hp.weight_shape + 0.5 * n * k_len,
                              1.0 / (hp.weight_rate + 0.5 * sw)), FLOOR)
    n_obs = int(pm.observed.sum())
    sr = ck.masked_sq_norm(r)
    st.gamma_eps = max(g5.gamma(hp.noise_shape + 0.5 * n_obs,
                                1.0 / (hp.noise_rate + 0.5 * sr)), FLOOR)
    if trace is not None:
        trace.update(sq_weights=sw, sq_resid=sr, n_obs=n_obs, m=st.usage.sum(axis=0))
    if not (math.isfinite(st.gamma_s) and math.isfinite(st.gamma_eps) and math.isfinite(sr)):
        raise DivergenceError(f"non-finite state at epoch {epoch}")
    st.epoch = epoch
    return st


def compose_estimates(st: State) -> np.ndarray:
    """bpfa.py:348-352."""
    out = np.empty((st.usage.shape[0], st.atoms.shape[1]), dtype=np.float64)
    ck.compose_estimates(st.usage, st.weights, st.atoms, out)
    return out


def infer(pm, hp, epochs, seed, freeze_dict=False, initial=None, init_mode="data",
          average_last=1, state=None, draws=None):
    """bpfa.py:379-414.  ``initial`` is an (atoms, pi) pair."""
    if epochs < 1:
        raise ValueError("epochs must be >= 1")
    if state is None:
        if initial is not None:
            state = install_dictionary(seed, pm, hp, initial[0], initial[1])
        else:
            state = init_state(pm, hp, seed, init_mode=init_mode)
    t_avg = max(1, min(int(average_last), epochs))
    acc = None
    for t in range(epochs):
        state = gibbs_epoch(state, pm, hp, freeze_dict=freeze_dict, draws=draws)
        if t >= epochs - t_avg:
            e = compose_estimates(state)
            acc = e if acc is None else acc + e
    return state, acc / t_avg
