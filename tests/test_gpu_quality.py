"""End-to-end reconstruction quality against the reference on identical inputs
(north_star correctness check 3; SURVEY §8c "PSNR within a stated ±0.1 dB, SSIM
within ±0.002").

The reference's PSNR / SSIM come from tests/golden/quality.json, produced by
running patchbeam itself on the same frames, masks and seeds
(tests/golden/make_quality.py; cases in tests/golden/quality_cases.py):

* replay mode (the reference's own draw streams, free-running): the device run
  of seed 0 must land within ±0.05 dB PSNR / ±0.001 SSIM of the reference's
  seed-0 run — configs[0] in full through the Python API, configs[2] (3 live
  512x512 frames) through the NATIVE problem (pb_problem_submit_frame), and the
  configs[1] crop;
* Philox mode (device draws — a different random stream of the same sampler):
  the mean over seeds 0, 1, 2 (and frames) must lie within ±0.1 dB PSNR /
  ±0.002 SSIM of the reference's mean over the same seeds.
"""

import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from quality_cases import SEEDS, reference_summary, run_device  # noqa: E402

pytestmark = pytest.mark.gpu

TOL_REPLAY_PSNR, TOL_REPLAY_SSIM = 0.05, 0.001
TOL_MEAN_PSNR, TOL_MEAN_SSIM = 0.1, 0.002


@pytest.fixture(scope="module")
def qref():
    return json.load(open(os.path.join(HERE, "golden", "quality.json")))


@pytest.mark.parametrize("name", ["cfg0", "cfg2", "cfg1crop"])
def test_replay_quality_matches_reference_seed0(qref, cuda_device, name):
    p_ref, s_ref = reference_summary(qref, name)
    got = np.array(run_device(name, SEEDS[0], rng="numpy"))
    print(name, "replay psnr", got[:, 0], "ref", p_ref[0], "ssim", got[:, 1], "ref", s_ref[0])
    assert np.abs(got[:, 0] - p_ref[0]).max() <= TOL_REPLAY_PSNR
    assert np.abs(got[:, 1] - s_ref[0]).max() <= TOL_REPLAY_SSIM


@pytest.mark.parametrize("name", ["cfg0", "cfg2", "cfg1crop"])
def test_philox_quality_mean_over_seeds_matches_reference(qref, cuda_device, name):
    p_ref, s_ref = reference_summary(qref, name)
    got = np.array([run_device(name, s, rng="philox") for s in SEEDS])   # (seeds, frames, 2)
    print(name, "philox psnr", got[..., 0].mean(), "ref", p_ref.mean(), "ssim", got[..., 1].mean(), "ref",
          s_ref.mean())
    assert abs(got[..., 0].mean() - p_ref.mean()) <= TOL_MEAN_PSNR
    assert abs(got[..., 1].mean() - s_ref.mean()) <= TOL_MEAN_SSIM


def test_replay_reconstruction_configs0_matches_reference(cuda_device):
    """The seed-0 configs[0] reconstruction itself (data consistency on), free-running
    replay over all 10 epochs.  f32 vs f64 arithmetic: a near-tie Z flip (≤ 2 per
    4 M draws per epoch, teacher-forced) changes that patch's later draws, so the
    free-running images agree closely but not exactly: the device image against
    the reference's at >= 60 dB PSNR (MSE <= 1e-6) and 99 % of the pixels within
    1e-3 (measured: 3e-7 without a flip; p99.9 1.3e-3, max 3.3e-3 with one)."""
    from paper_2311_15061_b200.metrics import psnr

    ref = np.load(os.path.join(HERE, "golden", "quality_cfg0_s0.npz"))["recon"]
    _, recs = run_device("cfg0", 0, rng="numpy", return_recon=True)
    d = np.abs(recs[0] - ref)
    print("cfg0 replay recon: max", d.max(), "p99", np.quantile(d, 0.99), "psnr vs ref", psnr(recs[0], ref))
    assert psnr(recs[0], ref) >= 60.0
    assert np.quantile(d, 0.99) <= 1e-3


def test_philox_sampler_unbiased_against_replay(cuda_device):
    """Device draws vs the reference's draws on the same configs[0] problem over
    8 seeds: the mean PSNR of the Philox sampler within 0.1 dB of the replay
    sampler's (which equals the reference per seed, test above).  Over 24 seeds
    the measured difference is -0.011 dB = 1.0 standard error
    (profiles/r02/philox_bias.txt)."""
    seeds = range(8)
    phi = np.array([run_device("cfg0", s, rng="philox")[0] for s in seeds])
    rep = np.array([run_device("cfg0", s, rng="numpy")[0] for s in seeds])
    d = phi[:, 0].mean() - rep[:, 0].mean()
    print("philox - replay", d, "dB")
    assert abs(d) <= TOL_MEAN_PSNR
    assert abs(phi[:, 1].mean() - rep[:, 1].mean()) <= TOL_MEAN_SSIM
