"""Teacher-forced replay parity helpers shared by the GPU parity tests and
tools/parity_stats.py (test infrastructure: imports the oracle as the checker).

Replay mode: both implementations consume the reference's own keyed draw
streams (bpfa.py:293-333).  Teacher forcing: every epoch starts from the
REFERENCE state of the previous epoch, so per-epoch differences are the device
sweep's own f32 error, not accumulated drift.  The reference states come from
the oracle, which is bit-exact to patchbeam (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import math

import numpy as np

from oracle import bpfa as ob
from oracle import patches as op
from paper_2311_15061_b200 import bpfa as gb
from paper_2311_15061_b200 import patches as pp

# Stated per-epoch tolerances (f32 device sweep vs the f64 reference, replay mode,
# teacher-forced).  SURVEY §8c measured an fp32 restatement at S <= 4e-6 rel,
# D <= 1.1e-6 abs and suggested S <= 1e-5 rel, D <= 1e-5 abs, flips <= 1e-6.
TOL_S_REL = 1e-5        # |dS| <= TOL_S_REL * max(1, |S|) on patches without a Z flip
TOL_D_ABS = 1e-5        # max |dD| over all atoms and pixels
TOL_PI_REL = 1e-6       # pi, when Z agrees (Beta draws from identical integer shapes)
TOL_GS_REL = 1e-6       # gamma_s, when Z agrees
TOL_GE_REL = 1e-4       # gamma_eps, when Z agrees (sum R^2 carries the f32 residual error)


def flip_budget(n, k):
    """Z flips allowed per epoch: near-ties of |logit(U) - log rho| only (SURVEY
    §8c: <= 1 per 4 M measured); stated as max(2, 1e-6 * N * K)."""
    return max(2, int(1e-6 * n * k))


class ArrayDraws:
    """oracle StreamDraws interface over pre-drawn (atom, code_u, code_g) arrays,
    so the oracle and the device consume the very same draw arrays."""

    def __init__(self, seed, atom, cu, cg):
        self.inner = ob.StreamDraws(seed)
        self.a, self.u, self.g = atom, cu, cg

    def atom(self, epoch, k, p_len):
        return self.a[k]

    def codes(self, epoch, k, n):
        return self.u[k], self.g[k]

    def pi_rng(self, epoch):
        return self.inner.pi_rng(epoch)

    def gamma_rng(self, epoch):
        return self.inner.gamma_rng(epoch)


def upload(st: ob.State, patch_shape):
    return gb.GibbsState.from_host(st.atoms, st.pi, st.usage, st.weights, st.gamma_s, st.gamma_eps,
                                   st.epoch, st.seed, patch_shape)


def compare(gstate, ref: ob.State):
    """Per-epoch error statistics of a device state against the reference's."""
    h = gstate.to_host()
    flips = h["usage"] != ref.usage
    ok = ~flips.any(axis=1)
    ds = np.abs(h["weights"][ok] - ref.weights[ok]) / np.maximum(1.0, np.abs(ref.weights[ok]))
    return dict(flips=int(flips.sum()), s_rel=float(ds.max(initial=0.0)),
                d_abs=float(np.abs(h["atoms"] - ref.atoms).max()),
                pi_rel=float((np.abs(h["pi"] - ref.pi) / np.maximum(np.abs(ref.pi), 1e-300)).max()),
                gs_rel=abs(h["weight_precision"] - ref.gamma_s) / ref.gamma_s,
                ge_rel=abs(h["noise_precision"] - ref.gamma_eps) / ref.gamma_eps,
                epoch_ok=h["epoch"] == ref.epoch)


def check(stats, n, k, name=""):
    assert stats["epoch_ok"], name
    assert stats["flips"] <= flip_budget(n, k), (name, "Z flips", stats)
    assert stats["s_rel"] <= TOL_S_REL, (name, "S", stats)
    assert stats["d_abs"] <= TOL_D_ABS, (name, "D", stats)
    if stats["flips"] == 0:
        assert stats["pi_rel"] <= TOL_PI_REL, (name, "pi", stats)
        assert stats["gs_rel"] <= TOL_GS_REL, (name, "gamma_s", stats)
        assert stats["ge_rel"] <= TOL_GE_REL, (name, "gamma_eps", stats)


def teacher_forced(img, mask, patch, k, epochs, seed, mean_subtract=True, init_mode="data", freeze=False,
                   initial=None, start=None, on_epoch=None):
    """Run `epochs` teacher-forced epochs; returns the list of per-epoch stats.

    The reference state of each epoch is the oracle's epoch from the previous
    reference state with the same draw arrays.  ``initial`` = (atoms, pi) installs
    a dictionary (bpfa.py:355-376); ``start`` = (oracle State) skips the init."""
    pm = pp.extract_patches(img, mask, pp.PatchSpec(patch), mean_subtract)
    opm = op.extract_patches(img, mask, patch, (), mean_subtract)
    hp = gb.Hyperparams(num_atoms=k)
    if start is not None:
        st = start
    elif initial is not None:
        st = ob.install_dictionary(seed, opm, hp, initial[0], initial[1])
    else:
        st = ob.init_state(opm, hp, seed, init_mode=init_mode)
    n = opm.values.shape[0]
    out = []
    for _ in range(epochs):
        e = st.epoch + 1
        atom, cu, cg = gb.reference_draws(seed, e, k, n, pm.patch_size, freeze)
        gs = upload(st, patch)
        gb.gibbs_epoch(gs, pm, hp, freeze_dict=freeze, rng="numpy", draws=(atom, cu, cg))
        ref = ob.gibbs_epoch(st.copy(), opm, hp, freeze_dict=freeze, draws=ArrayDraws(seed, atom, cu, cg))
        s = compare(gs, ref)
        s["epoch"] = e
        out.append(s)
        if on_epoch is not None:
            on_epoch(s)
        st = ref
        del gs
    return out, (pm, opm, st)


def fmt(stats):
    return (f"e{stats['epoch']}: flips {stats['flips']} S {stats['s_rel']:.2e} D {stats['d_abs']:.2e} "
            f"pi {stats['pi_rel']:.2e} gs {stats['gs_rel']:.2e} ge {stats['ge_rel']:.2e}")


__all__ = ["teacher_forced", "check", "compare", "upload", "ArrayDraws", "fmt", "flip_budget", "math"]
