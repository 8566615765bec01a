"""GPU parity of the Gibbs sweep against the oracle (pinned bit-exact to the
reference by tests/test_oracle_golden.py).

Stated tolerances (f32 device state vs the reference's f64):
  * replay ("numpy") mode, teacher-forced per epoch from the reference state:
      the constants of tests/_parity.py — S <= 1e-5 rel (|dS| <= 1e-5 * max(1,|S|)
      on patches without a Z flip), atoms |dD| <= 1e-5 abs, pi / gamma_s <= 1e-6
      rel and gamma_eps <= 1e-4 rel when Z agrees, Z flips <= max(2, 1e-6 N K);
  * kernel seam (residual / code_moments / atom_moments / compose): rel 1e-5;
  * free-running PSNR within 0.1 dB of the reference trajectory.
"""

import math

import numpy as np
import pytest
import torch

from _parity import check, compare, fmt
from oracle import bpfa as ob
from oracle import patches as op
from paper_2311_15061_b200 import bpfa as gb
from paper_2311_15061_b200 import patches as pp

pytestmark = pytest.mark.gpu


def _pm_pair(img, mask, patch, ms):
    return (pp.extract_patches(img, mask, pp.PatchSpec(patch), ms),
            op.extract_patches(img, mask, patch, (), ms))


def _upload(st: ob.State, patch_shape):
    return gb.GibbsState.from_host(st.atoms, st.pi, st.usage, st.weights, st.gamma_s, st.gamma_eps,
                                   st.epoch, st.seed, patch_shape)


def _random_state(opm, k, seed):
    rng = np.random.default_rng(seed)
    n, p = opm.values.shape
    return ob.State(atoms=rng.standard_normal((k, p)) * 0.3, pi=rng.uniform(0.05, 0.95, k),
                    usage=rng.random((n, k)) < 0.5, weights=rng.standard_normal((n, k)),
                    gamma_s=float(rng.uniform(0.5, 4.0)), gamma_eps=float(rng.uniform(0.5, 50.0)),
                    epoch=0, seed=seed)


def test_seam_kernels_match_oracle(cuda_device):
    rng = np.random.default_rng(3)
    img = rng.random((40, 37))
    mask = rng.random(img.shape) < 0.3
    for patch in ((8, 8), (10, 10), (3, 3), (16, 16)):
        pm, opm = _pm_pair(img, mask, patch, True)
        st = _random_state(opm, 7, 11)
        gs = _upload(st, patch)
        r_gpu = gb._residual(pm, gs).T.double().cpu().numpy()
        r_ref = ob.residual(opm, st)
        assert np.abs(r_gpu - r_ref).max() <= 1e-5 * max(1.0, np.abs(r_ref).max()), patch
        est = gb.compose_estimates(gs).double().cpu().numpy()
        assert np.abs(est - ob.compose_estimates(st)).max() <= 1e-5 * max(1.0, np.abs(est).max())
        for k in (0, 3, 6):
            lam, mu = gb.atom_posterior(pm, gs, k)
            olam, omu = ob.atom_posterior(opm, st, k)
            assert np.allclose(lam, olam, rtol=1e-5, atol=1e-5)
            assert np.allclose(mu, omu, rtol=1e-4, atol=1e-5)
            lr, al, me = gb.code_posterior(pm, gs, k)
            olr, oal, ome = ob.code_posterior(opm, st, k)
            assert np.allclose(al, oal, rtol=1e-5)
            assert np.allclose(me, ome, rtol=1e-4, atol=1e-5)
            assert np.allclose(lr, olr, rtol=1e-4, atol=1e-3)
        a, b = gb.pi_posterior(gs, ob.Hyper(num_atoms=7))
        oa, obb = ob.pi_posterior(st, ob.Hyper(num_atoms=7))
        assert np.array_equal(a, oa) and np.array_equal(b, obb)
        hp = gb.Hyperparams(num_atoms=7)
        (ws, wr), (ns, nr) = gb.gamma_posteriors(pm, gs, hp)
        (ows, owr), (ons, onr) = ob.gamma_posteriors(opm, st, hp)
        assert ws == ows and ns == ons
        assert math.isclose(wr, owr, rel_tol=1e-5) and math.isclose(nr, onr, rel_tol=1e-4)


def _compare_epoch(name, gstate, ref: ob.State, n, k):
    st = compare(gstate, ref)
    print(name, fmt(dict(st, epoch=ref.epoch)))
    check(st, n, k, name)
    return st["flips"]


@pytest.mark.parametrize("name", ["small", "linehop", "cfg1crop", "frozen", "avg", "cube"])
def test_teacher_forced_epochs_replay_mode(golden, cuda_device, name):
    """Each epoch starts from the REFERENCE state; both sides consume the
    reference's own draw streams (replay mode)."""
    g = golden(f"traj_{name}.npz")
    patch = tuple(int(b) for b in g["patch"])
    ms = bool(g["mean_subtract"])
    pm, opm = _pm_pair(g["img"], g["mask"], patch, ms)
    hp = gb.Hyperparams(num_atoms=int(g["k"]))
    seed = int(g["seed"])
    freeze = bool(g["freeze"])
    if "init_atoms" in g:
        st = ob.install_dictionary(seed, opm, hp, g["init_atoms"], g["init_pi"])
    else:
        st = ob.init_state(opm, hp, seed, init_mode=str(g["init_mode"]))
    n, k = st.usage.shape
    total = 0
    for e in range(1, int(g["epochs"]) + 1):
        gs = _upload(st, patch)
        gb.gibbs_epoch(gs, pm, hp, freeze_dict=freeze, rng="numpy")
        ref = ob.State(atoms=g[f"e{e}_atoms"], pi=g[f"e{e}_pi"], usage=g[f"e{e}_usage"],
                       weights=g[f"e{e}_weights"], gamma_s=float(g[f"e{e}_gammas"][0]),
                       gamma_eps=float(g[f"e{e}_gammas"][1]), epoch=e, seed=seed)
        total += _compare_epoch(f"{name}/e{e}", gs, ref, n, k)
        st = ref.copy()
    print(f"{name}: total Z flips {total}")


def test_init_state_matches_reference(golden, cuda_device):
    g = golden("traj_cfg1crop.npz")
    pm = pp.extract_patches(g["img"], g["mask"], pp.PatchSpec((8, 8)), True)
    st = gb.init_state(pm, gb.Hyperparams(num_atoms=int(g["k"])), int(g["seed"]), "data")
    assert np.abs(st.dictionary.atoms.double().cpu().numpy() - g["e0_atoms"]).max() <= 1e-6
    assert st.epoch == 0 and st.weight_precision == 1.0 and st.noise_precision == 1.0


def test_free_running_psnr_parity_replay(golden, cuda_device):
    """Full infer (reference draw streams) -> reconstruction PSNR within 0.1 dB."""
    from paper_2311_15061_b200.metrics import psnr

    g = golden("traj_cfg1crop.npz")
    pm = pp.extract_patches(g["img"], g["mask"], pp.PatchSpec((8, 8)), True)
    hp = gb.Hyperparams(num_atoms=int(g["k"]))
    _, est = gb.infer(pm, hp, int(g["epochs"]), int(g["seed"]), rng="numpy")
    rec = pp.reconstitute(pm, est, dc_original=g["img"], dc_mask=g["mask"])
    ref_psnr = psnr(g["recon_dc"], g["img"])
    assert abs(psnr(rec, g["img"]) - ref_psnr) <= 0.1, (psnr(rec, g["img"]), ref_psnr)


def test_philox_z_marginal_frequency(cuda_device):
    """Criterion 6 (test_acceptance.py:192-225) as one data-parallel launch:
    20,000 identical single-patch problems, one draw each; frequency of z=1
    within 3 sigma of sigmoid(log_rho)."""
    draws = 20000
    atom = np.array([0.6, -0.2, 0.4, 0.1])
    rng = np.random.default_rng(5)
    img = rng.random((2, 2))
    tiled = np.tile(img, (1, draws))            # draws disjoint 2x2 blocks side by side
    pm = pp.extract_patches(tiled, np.ones_like(tiled, bool), pp.PatchSpec((2, 2), (2, 2)))
    assert pm.num_patches == draws
    hp = gb.Hyperparams(num_atoms=1)
    st = gb.GibbsState.from_host(atom[None, :], [0.35], np.ones((draws, 1), bool), np.full((draws, 1), 0.8),
                                 2.0, 5.0, 0, 7, (2, 2))
    gb.gibbs_epoch(st, pm, hp, freeze_dict=True, rng="philox", check=False)
    hits = int(st.usage_kn.sum().item())
    opm = op.extract_patches(img, np.ones((2, 2), bool), (2, 2), (), False)
    ost = ob.State(atoms=atom[None, :].copy(), pi=np.array([0.35]), usage=np.ones((1, 1), bool),
                   weights=np.full((1, 1), 0.8), gamma_s=2.0, gamma_eps=5.0, epoch=0, seed=7)
    lr, _, _ = ob.code_posterior(opm, ost, 0)
    p1 = 1.0 / (1.0 + math.exp(-float(lr[0])))
    sigma = math.sqrt(p1 * (1 - p1) / draws)
    assert abs(hits / draws - p1) <= 3 * sigma, (hits / draws, p1)


def test_masked_update_invariance_and_determinism(cuda_device):
    from paper_2311_15061_b200 import inputs

    rng = np.random.default_rng(8)
    img = rng.random((24, 24))
    mask = inputs.make_mask(img.shape, 0.5, "uniform-random", 9)
    garbage = img.copy()
    garbage[~mask] = rng.random((~mask).sum()) * 100 - 50
    hp = gb.Hyperparams(num_atoms=6)
    outs = []
    for data in (img, garbage, img):
        pm = pp.extract_patches(data, mask, pp.PatchSpec((4, 4)), True)
        st, est = gb.infer(pm, hp, epochs=3, seed=10, rng="philox")
        outs.append((est.cpu(), st.dictionary.atoms.cpu(), st.weights_kn.cpu(), st.noise_precision))
    for o in outs[1:]:
        assert torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1]) and torch.equal(o[2], outs[0][2])
        assert o[3] == outs[0][3]
    pm = pp.extract_patches(img, mask, pp.PatchSpec((4, 4)), True)
    _, est_c = gb.infer(pm, hp, epochs=3, seed=11, rng="philox")
    assert not torch.equal(est_c.cpu(), outs[0][0])


def test_epoch_counting_and_freeze(cuda_device):
    rng = np.random.default_rng(7)
    img = rng.random((10, 10))
    pm = pp.extract_patches(img, rng.random((10, 10)) < 0.5, pp.PatchSpec((3, 3)))
    hp = gb.Hyperparams(num_atoms=4)
    st, _ = gb.infer(pm, hp, epochs=2, seed=1)
    assert st.epoch == 2
    fr = gb.init_state(pm, hp, seed=2, init_mode="data")
    before = fr.dictionary.atoms.clone()
    for _ in range(3):
        gb.gibbs_epoch(fr, pm, hp, freeze_dict=True)
    assert torch.equal(fr.dictionary.atoms, before) and fr.epoch == 3


def test_divergence_detection(cuda_device):
    rng = np.random.default_rng(21)
    img = rng.random((6, 6))
    pm = pp.extract_patches(img, rng.random((6, 6)) < 0.5, pp.PatchSpec((2, 2)))
    hp = gb.Hyperparams(num_atoms=2)
    for mode in ("philox", "numpy"):
        st = gb.init_state(pm, hp, seed=22, init_mode="prior")
        st.weights[:] = float("inf")
        st.usage[:] = True
        with pytest.raises(gb.DivergenceError):
            gb.gibbs_epoch(st, pm, hp, rng=mode)


def test_frozen_known_atom_regression(cuda_device):
    rng = np.random.default_rng(12)
    patch = rng.random((3, 3))
    d = gb.Dictionary(atoms=(patch.ravel() / np.linalg.norm(patch))[None, :].copy(), pi=np.array([0.9]),
                      patch_shape=(3, 3))
    pm = pp.extract_patches(patch, np.ones((3, 3), bool), pp.PatchSpec((3, 3)))
    hp = gb.Hyperparams(num_atoms=1, noise_shape=1e8, noise_rate=1e2, weight_shape=1e-2, weight_rate=1e-2)
    for mode in ("philox", "numpy"):
        _, est = gb.infer(pm, hp, epochs=20, seed=13, freeze_dict=True, initial_dict=d, rng=mode)
        assert float(((est[0].double().cpu().numpy() - patch.ravel()) ** 2).mean()) < 1e-4


def test_synthetic_dictionary_recovery_beats_mean_fill(cuda_device):
    """test_bpfa.py:264-293 on the device (philox mode)."""
    rng = np.random.default_rng(14)
    k_true, p_len, n = 4, 25, 300
    true_atoms = rng.standard_normal((k_true, p_len))
    true_atoms /= np.linalg.norm(true_atoms, axis=1, keepdims=True)
    w = rng.standard_normal((n, k_true)) * (rng.random((n, k_true)) < 0.6)
    clean = w @ true_atoms
    observed = rng.random((n, p_len)) < 0.5
    # lay the n patches out as disjoint 5x5 tiles of a (5, 5n) image
    img = clean.reshape(n, 5, 5).transpose(1, 0, 2).reshape(5, 5 * n)
    msk = observed.reshape(n, 5, 5).transpose(1, 0, 2).reshape(5, 5 * n)
    pm = pp.extract_patches(img, msk, pp.PatchSpec((5, 5), (5, 5)))
    _, est = gb.infer(pm, gb.Hyperparams(num_atoms=8), epochs=30, seed=15)
    est = est.double().cpu().numpy()
    held = ~observed
    model = float(np.mean((est[held] - clean[held]) ** 2))
    cnt = observed.sum(1, keepdims=True)
    fill = np.where(cnt > 0, (np.where(observed, clean, 0).sum(1, keepdims=True) / np.maximum(cnt, 1)), 0)
    base = float(np.mean((np.broadcast_to(fill, clean.shape)[held] - clean[held]) ** 2))
    assert model < 0.1 * base, (model, base)


def test_residual_carry_matches_recompute(cuda_device):
    """Carrying the end-of-sweep residual into the next epoch (PB_RESID_CARRY)
    equals recomputing residual_full each epoch (the reference's behaviour,
    bpfa.py:297) up to f32 rounding drift; the R = X start of fresh codes is exact."""
    from paper_2311_15061_b200 import inputs

    img = inputs.synthetic_texture((48, 48), seed=2)
    mask = inputs.make_mask(img.shape, 0.25, "uniform-random", 2)
    hp = gb.Hyperparams(num_atoms=12)
    pm = pp.extract_patches(img, mask, pp.PatchSpec((8, 8)), True)
    a = gb.init_state(pm, hp, 5, "prior")
    b = gb.init_state(pm, hp, 5, "prior")
    for _ in range(4):
        gb.gibbs_epoch(a, pm, hp, rng="philox", check=False)       # carry after the first epoch
        b._resid_key = None
        b._zero_key = None if b.epoch > 0 else b._zero_key
        gb.gibbs_epoch(b, pm, hp, rng="philox", check=False)       # forced recompute
    ha, hb = a.to_host(), b.to_host()
    assert (ha["usage"] != hb["usage"]).sum() <= 2
    ok = ~(ha["usage"] != hb["usage"]).any(axis=1)
    assert np.abs(ha["weights"][ok] - hb["weights"][ok]).max() <= 1e-3
    assert np.abs(ha["atoms"] - hb["atoms"]).max() <= 1e-4


@pytest.mark.parametrize("rng", ["philox", "numpy"])
def test_zero_codes_dictionary_step_is_prior_redraw(cuda_device, rng):
    """With Z*S == 0 (fresh init, warm-reset live frame) the dictionary step is
    the prior redraw d_k = g/sqrt(P).  The short path
    (k_dict_prior, taken when the codes are known to be zero) must give the same
    state, bit for bit, as the full K/8-pass kernel run on the same zero codes."""
    from paper_2311_15061_b200 import inputs

    img = inputs.synthetic_texture((64, 64), seed=4)
    mask = inputs.make_mask(img.shape, 0.25, "uniform-random", 4)
    hp = gb.Hyperparams(num_atoms=20)
    pm = pp.extract_patches(img, mask, pp.PatchSpec((8, 8)), True)
    a = gb.init_state(pm, hp, 11, "data")
    b = gb.init_state(pm, hp, 11, "data")
    b._zero_key = None                       # not known to be zero: residual_full + full dictionary step
    for _ in range(2):
        gb.gibbs_epoch(a, pm, hp, rng=rng, check=False)
        gb.gibbs_epoch(b, pm, hp, rng=rng, check=False)
        ha, hb = a.to_host(), b.to_host()
        for key in ("atoms", "usage", "weights", "pi"):
            assert np.array_equal(ha[key], hb[key]), key
        assert ha["weight_precision"] == hb["weight_precision"]
        assert ha["noise_precision"] == hb["noise_precision"]


def test_infer_average_last_matches_reference(golden, cuda_device):
    """infer(average_last=2) in replay mode against the reference's tail-averaged
    estimate (traj_avg.npz: bpfa.py:379-414 with average_last=2, prior init, no
    mean subtraction): same draws, free-running, estimates within 1e-4."""
    g = golden("traj_avg.npz")
    patch = tuple(int(b) for b in g["patch"])
    pm = pp.extract_patches(g["img"], g["mask"], pp.PatchSpec(patch), bool(g["mean_subtract"]))
    hp = gb.Hyperparams(num_atoms=int(g["k"]))
    st, est = gb.infer(pm, hp, int(g["epochs"]), int(g["seed"]), init_mode=str(g["init_mode"]),
                       average_last=int(g["average_last"]), rng="numpy")
    h = st.to_host()
    assert np.array_equal(h["usage"], g[f"e{int(g['epochs'])}_usage"])
    err = np.abs(est.double().cpu().numpy() - g["est"]).max()
    assert err <= 1e-4, err
    rec = pp.reconstitute(pm, est)
    assert np.abs(rec - g["recon"]).max() <= 1e-4


@pytest.mark.parametrize("case", ["p64k16", "p100k256"])
def test_epoch_statistics_large_problem_claimed_code_step(cuda_device, case):
    """Problems past 2^17 patches run the warp-claimed code step; at P = 100,
    K = 256 (configs[1]'s shape) it is combined with the pitch-8 swizzled w
    windows.  The epoch's sum S^2, sum R^2 and usage counts m_k equal host
    recomputations from the resulting state (f32 accumulation noise only)."""
    if case == "p64k16":
        shape, patch, k = (1032, 1032), (8, 8), 16     # > 2^20 patches: two-level finish
    else:
        shape, patch, k = (420, 420), (10, 10), 256    # 168,921 patches >= 2^17
    from paper_2311_15061_b200 import inputs

    img = inputs.synthetic_texture(shape, seed=6)
    mask = inputs.make_mask(shape, 0.1, "uniform-random", 6)
    hp = gb.Hyperparams(num_atoms=k)
    pm = pp.extract_patches(img, mask, pp.PatchSpec(patch), True)
    assert pm.num_patches >= 1 << 17
    st = gb.init_state(pm, hp, 3, "prior")
    for _ in range(2):   # (the usage counts m_k of the last epoch stay in the state's workspace)
        gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
    m = st.workspace(pm.num_patches, pm.patch_size, k, pm.n_obs)[1]
    s = st._sc()
    w = st.weights_kn[:, :pm.num_patches].double()
    assert abs(s.sq_w - float((w * w).sum())) <= 1e-6 * s.sq_w
    r = gb._residual(pm, st).double()
    assert abs(s.sq_r - float((r * r).sum())) <= 1e-3 * s.sq_r
    mk = st.usage_kn[:, :pm.num_patches].sum(dim=1, dtype=torch.int64).cpu().numpy()
    assert np.array_equal(m.cpu().numpy().astype(np.int64), mk)

