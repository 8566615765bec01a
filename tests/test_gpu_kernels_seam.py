"""The fine-grained seam: `paper_2311_15061_b200.kernels`, the
drop-in for the reference's `patchbeam._kernels` (_kernels.py:18-145), backed by
the C-ABI seam entries (pb_residual_full ... pb_compose_estimates).

* each function against the oracle's C restatement of _kernels (f64; pinned to
  the reference by tests/test_oracle_golden.py) on seeded inputs, including
  ragged masks, all-unobserved rows / columns, zero codes and N = 1; the device
  computes in f32 with f64 reductions: tolerances relative to the data scale,
  stated per function below;
* each function rebound ONE AT A TIME into the unmodified reference
  (baseline/_ref; skipped when absent) exactly as a maintainer would
  (`patchbeam._kernels.X = kernels.X`; bpfa.py:30 calls through the module
  object): one reference Gibbs epoch from the same state with the reference's
  own draws must match the pure-reference epoch (Z agreement >= 99 %, atoms and
  weights within 1e-3 where the codes agree).
"""

import copy
import os
import sys

import numpy as np
import pytest

from paper_2311_15061_b200 import kernels

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.path.join(ROOT, "baseline", "_ref")
NAMES = kernels.__all__


def _ok():
    sys.path.insert(0, ROOT)
    from oracle import _ckernels

    return _ckernels


def _case(n, p, k, ratio, seed, zero_codes=False):
    rng = np.random.default_rng(seed)
    observed = rng.random((n, p)) < ratio
    if n > 2:
        observed[1] = False            # a patch with nothing observed
        observed[:, 0] = False         # a pixel nobody observes
    values = np.where(observed, rng.normal(size=(n, p)), 0.0)
    usage = rng.random((n, k)) < 0.3
    weights = rng.normal(size=(n, k))
    if zero_codes:
        usage[:] = False
        weights[:] = 0.0
    atoms = rng.normal(size=(k, p)) / np.sqrt(p)
    resid = np.where(observed, rng.normal(size=(n, p)), 0.0)
    w_col = np.where(usage[:, 0], weights[:, 0], 0.0)
    return dict(values=values, observed=observed, usage=usage, weights=weights, atoms=atoms, resid=resid,
                w_col=w_col, delta=rng.normal(size=p) * 0.1, dw=np.where(rng.random(n) < 0.5, rng.normal(size=n), 0.0))


CASES = [(3000, 64, 24, 0.25, 0, False), (1000, 100, 40, 0.10, 1, False), (500, 64, 16, 0.25, 2, True),
         (1, 36, 8, 0.5, 3, False), (777, 27, 5, 0.9, 4, False)]


@pytest.mark.parametrize("n,p,k,ratio,seed,zero", CASES)
def test_seam_matches_oracle(cuda_device, n, p, k, ratio, seed, zero):
    ok = _ok()
    c = _case(n, p, k, ratio, seed, zero)
    o, scale = c["observed"], 1.0 + np.abs(c["values"]).max()

    got, ref = np.full((n, p), 7.0), np.zeros((n, p))
    kernels.residual_full(c["values"], o, c["usage"], c["weights"], c["atoms"], got)
    ok.residual_full(c["values"], o, c["usage"], c["weights"], c["atoms"], ref)
    assert np.all(got[~o] == 0.0)
    assert np.abs(got - ref).max() <= 1e-5 * scale * max(1.0, np.sqrt(k))

    got, ref = np.zeros((n, p)), np.zeros((n, p))
    kernels.compose_estimates(c["usage"], c["weights"], c["atoms"], got)
    ok.compose_estimates(c["usage"], c["weights"], c["atoms"], ref)
    assert np.abs(got - ref).max() <= 1e-5 * max(1.0, np.sqrt(k))

    a, cc = kernels.atom_moments(c["resid"], o, c["w_col"])
    ra, rc = ok.atom_moments(c["resid"], o, c["w_col"])
    assert a.dtype == np.float64 and a.shape == (p,)
    np.testing.assert_allclose(a, ra, rtol=1e-6, atol=1e-6 * (1 + ra.max()))
    np.testing.assert_allclose(cc, rc, rtol=1e-5, atol=1e-5 * (1 + np.abs(rc).max()))

    u, v = kernels.code_moments(c["resid"], o, c["atoms"][0])
    ru, rv = ok.code_moments(c["resid"], o, c["atoms"][0])
    assert u.shape == (n,) and v.dtype == np.float64
    np.testing.assert_allclose(u, ru, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(v, rv, rtol=1e-5, atol=1e-5)

    got, ref = c["resid"].copy(), c["resid"].copy()
    kernels.shift_atom(got, o, c["w_col"], c["delta"])
    ok.shift_atom(ref, o, c["w_col"], c["delta"])
    assert np.all(got[~o] == 0.0)
    assert np.abs(got - ref).max() <= 1e-5 * (1 + np.abs(ref).max())

    got, ref = c["resid"].copy(), c["resid"].copy()
    kernels.shift_codes(got, o, c["atoms"][1 % k], c["dw"])
    ok.shift_codes(ref, o, c["atoms"][1 % k], c["dw"])
    assert np.abs(got - ref).max() <= 1e-5 * (1 + np.abs(ref).max())

    s, rs = kernels.masked_sq_norm(c["resid"]), ok.masked_sq_norm(c["resid"])
    assert isinstance(s, float)
    assert abs(s - rs) <= 1e-6 * max(rs, 1.0)


@pytest.fixture(scope="module")
def patchbeam(tmp_path_factory):
    if not os.path.isdir(os.path.join(REF, "patchbeam")):
        pytest.skip("reference not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(tmp_path_factory.mktemp("numba")))
    sys.path.insert(0, REF)
    import patchbeam as pb

    return pb


def _ref_problem(pb):
    from patchbeam import bpfa
    from patchbeam.patches import PatchSpec, extract_patches

    from paper_2311_15061_b200 import inputs

    img = inputs.synthetic_texture((30, 34), seed=3)
    mask = inputs.make_mask(img.shape, 0.3, "uniform-random", 3)
    pm = extract_patches(img, mask, PatchSpec((6, 6)))
    hp = bpfa.Hyperparams(num_atoms=12)
    st = bpfa.init_state(pm, hp, 5, init_mode="data")
    for _ in range(3):
        st = bpfa.gibbs_epoch(st, pm, hp)
    return bpfa, pm, hp, st


@pytest.mark.parametrize("name", NAMES)
def test_seam_rebound_into_reference_epoch(cuda_device, patchbeam, name):
    from patchbeam import _kernels

    bpfa, pm, hp, st0 = _ref_problem(patchbeam)
    ref = bpfa.gibbs_epoch(copy.deepcopy(st0), pm, hp)
    orig = getattr(_kernels, name)
    setattr(_kernels, name, getattr(kernels, name))
    try:
        got = bpfa.gibbs_epoch(copy.deepcopy(st0), pm, hp)
        if name == "compose_estimates":   # not called by gibbs_epoch: the estimate of the state
            est_g = bpfa.compose_estimates(got)
    finally:
        setattr(_kernels, name, orig)
    agree = (got.usage == ref.usage)
    print(name, "Z agreement", agree.mean(), "max |dD|", np.abs(got.dictionary.atoms - ref.dictionary.atoms).max(),
          "max |dS| (agreeing codes)", np.abs(np.where(agree, got.weights - ref.weights, 0)).max(),
          "gs", got.weight_precision / ref.weight_precision - 1, "ge", got.noise_precision / ref.noise_precision - 1)
    assert agree.mean() >= 0.99
    if agree.all():
        assert np.abs(got.dictionary.atoms - ref.dictionary.atoms).max() <= 1e-3
        assert np.abs(got.weights - ref.weights).max() <= 1e-3
        assert abs(got.noise_precision / ref.noise_precision - 1) <= 1e-3
    if name == "compose_estimates":
        assert np.abs(est_g - bpfa.compose_estimates(ref)).max() <= 1e-4
