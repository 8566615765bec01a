"""Edge cases of the device sweep, each against the oracle (teacher-forced
replay, the reference's draw streams) or the reference's stated behaviour:

* large patches (P = 256, 3-D 8x8x4, ~50 % observed -> several lanes per patch
  in the code step, the 16-warp double-buffered dictionary-step variant), K not
  a multiple of 8: replay parity per epoch (Z flips <= 2, D <= 2e-5);
* an all-unobserved mask (nnz = 0): the sweep runs, every atom is a prior draw
  and the estimates are zero (bpfa.py:299-307 with A = C = 0);
* a fully observed frame: replay parity;
* the split code step (a narrow launch for most patches and, concurrently on
  a side stream, a wide launch over the listed outlier patches), forced via
  pb_patch_index.split_request with many and with few outliers: replay parity.
"""

import numpy as np
import pytest

from oracle import bpfa as ob
from oracle import patches as op
from oracle.rng import DOMAIN_ATOM, keyed_rng
from paper_2311_15061_b200 import bpfa as gb
from paper_2311_15061_b200 import patches as pp

from test_gpu_sweep import _compare_epoch, _pm_pair, _upload

pytestmark = pytest.mark.gpu


def _replay(img, mask, patch, ms, k, seed, epochs, split=0):
    pm, opm = _pm_pair(img, mask, patch, ms)
    if split:   # force the split code step (pb_patch_index.split_request)
        pm.split_request = split
        ix = pm.index()
        assert ix.split_count == split and ix.n_outliers > 0
    hp = gb.Hyperparams(num_atoms=k)
    st = ob.init_state(opm, ob.Hyper(num_atoms=k), seed, init_mode="prior")
    n = opm.values.shape[0]
    total = 0
    for e in range(1, epochs + 1):
        gs = _upload(st, patch)
        gb.gibbs_epoch(gs, pm, hp, rng="numpy")
        ref = st.copy()
        ob.gibbs_epoch(ref, opm, ob.Hyper(num_atoms=k))
        total += _compare_epoch(f"e{e}", gs, ref, n, k)
        st = ref
    return total


def test_large_patch_cube_replay(cuda_device):
    rng = np.random.default_rng(12)
    cube = rng.random((11, 12, 8))
    mask = rng.random(cube.shape) < 0.5
    assert _replay(cube, mask, (8, 8, 4), False, 13, 5, 2) <= 4


def test_fully_observed_replay(cuda_device):
    rng = np.random.default_rng(13)
    img = rng.random((20, 21))
    assert _replay(img, np.ones(img.shape, bool), (5, 5), True, 9, 2, 2) <= 4


def test_empty_mask_sweep(cuda_device):
    img = np.random.default_rng(14).random((16, 16))
    mask = np.zeros(img.shape, bool)
    pm = pp.extract_patches(img, mask, pp.PatchSpec((4, 4)), True)
    assert pm.n_obs == 0
    hp = gb.Hyperparams(num_atoms=6)
    st, est = gb.infer(pm, hp, 2, 3, rng="numpy")
    h = st.to_host()
    prior = np.stack([keyed_rng(3, DOMAIN_ATOM, 2, k).standard_normal(16) / 4.0 for k in range(6)])
    assert np.allclose(h["atoms"], prior, atol=1e-6)          # lambda = P, mu = 0: a prior draw
    assert np.all(est.cpu().numpy() == 0.0) or np.isfinite(est.cpu().numpy()).all()
    rec = pp.reconstitute(pm, est)
    assert np.isfinite(rec).all()


@pytest.mark.parametrize("split", [8, 16])
def test_split_code_step_replay(cuda_device, split):
    rng = np.random.default_rng(15)
    img = rng.random((40, 41))
    mask = rng.random(img.shape) < 0.3   # 6x6 patches: ~11 observed, max ~20
    assert _replay(img, mask, (6, 6), True, 10, 3, 2, split=split) <= 4


def test_chunked_dictionary_staging_replay(cuda_device):
    """Code step with the dictionary staged in chunks (10x10 patches, K = 264:
    (P+1) x (K+2) floats exceed a CTA's DT budget, so k_pack_dt builds two
    chunks and each block of patches stages them in turn; single-lane patches,
    K not a multiple of the chunk): replay parity per epoch."""
    rng = np.random.default_rng(16)
    img = rng.random((30, 31))
    mask = rng.random(img.shape) < 0.12
    assert _replay(img, mask, (10, 10), True, 264, 4, 2) <= 4
