"""The train / inpaint entry flows (reference cli.py) on the device against
the reference's own outputs (tests/golden/entry.npz, produced by patchbeam):

* normalize_observed (cli.py:195-212): bit-exact values, scale and offset;
* inpaint (cmd_inpaint's steps, replay mode): reconstruction within 1e-4,
  dictionary within 1e-5;
* learn (cmd_learn's steps: masks keyed by seed + i, concatenated patch
  matrices, replay mode): dictionary within 1e-5, pi within 1e-6;
* transfer_dictionary onto an extended patch shape (bpfa.py:417-458) on the
  device: within 1e-6 (f32 output of f32-exact atoms);
* the live problem: installing a dictionary of another atom count, and
  Pipeline.transfer_between (pipeline.py:294-304) from a 2-D problem onto a
  cube problem, device to device.
"""

import numpy as np
import pytest
import torch

from paper_2311_15061_b200 import bpfa as gb
from paper_2311_15061_b200 import entry
from paper_2311_15061_b200 import inputs
from paper_2311_15061_b200 import patches as pp
from paper_2311_15061_b200.live import LiveProblem, transfer_between

pytestmark = pytest.mark.gpu


def test_normalize_observed_bit_exact(golden, cuda_device):
    g = golden("entry.npz")
    for i in range(4):
        out, sc, off = entry.normalize_observed(g[f"n{i}_frame"], g[f"n{i}_mask"])
        assert np.array_equal(out, g[f"n{i}_out"]), i
        assert (sc, off) == tuple(g[f"n{i}_scale_offset"]), i
        dev, sc2, off2 = entry.normalize_observed(torch.as_tensor(g[f"n{i}_frame"]).cuda(),
                                                  torch.as_tensor(g[f"n{i}_mask"]).cuda())
        assert dev.is_cuda and (sc2, off2) == (sc, off)


def test_inpaint_flow_matches_reference(golden, cuda_device):
    g = golden("entry.npz")
    r = entry.inpaint(g["inp_img"], g["inp_mask"], pp.PatchSpec((5, 5)), gb.Hyperparams(num_atoms=12), epochs=3,
                      seed=4, rng="numpy")
    assert (r.scale, r.offset) == tuple(g["inp_scale_offset"])
    assert np.abs(r.reconstruction - g["inp_recon"]).max() <= 1e-4
    assert np.abs(r.state.dictionary.atoms.double().cpu().numpy() - g["inp_atoms"]).max() <= 1e-5


def test_learn_flow_matches_reference(golden, cuda_device, tmp_path):
    from paper_2311_15061_b200.formats import read_dict

    g = golden("entry.npz")
    out = tmp_path / "d.sadf"
    r = entry.learn([g["learn_img0"], g["learn_img1"]], pp.PatchSpec((4, 4)), num_atoms=7, epochs=3, seed=5,
                    mask_ratio=0.35, rng="numpy", dict_out=str(out))
    assert r.num_patches == int(g["learn_n"])
    assert np.abs(r.dictionary.atoms.double().cpu().numpy() - g["learn_atoms"]).max() <= 1e-5
    assert np.abs(r.dictionary.pi.cpu().numpy() - g["learn_pi"]).max() <= 1e-6
    d = read_dict(str(out))
    assert d.atoms.shape == (7, 16) and tuple(d.patch_shape) == (4, 4)


def test_transfer_dictionary_on_device(golden, cuda_device):
    g = golden("entry.npz")
    src = gb.Dictionary(g["tr_src"].copy(), g["tr_pi"].copy(), (3, 4))
    host = gb.transfer_dictionary(src, (3, 4, 3), (10, 12, 3))
    assert host.atoms.shape == (5, 36) and np.abs(host.atoms - g["tr_out"]).max() <= 1e-6
    dev = gb.transfer_dictionary(gb.Dictionary(torch.as_tensor(g["tr_src"], dtype=torch.float32).cuda(),
                                               torch.as_tensor(g["tr_pi"]).cuda(), (3, 4)), (3, 4, 3))
    assert dev.atoms.is_cuda and np.abs(dev.atoms.double().cpu().numpy() - g["tr_out"]).max() <= 1e-6
    same = gb.transfer_dictionary(src, (3, 4))
    assert np.array_equal(same.atoms, src.atoms)
    with pytest.raises(pp.ShapeError):
        gb.transfer_dictionary(src, (3, 5, 2))
    with pytest.raises(pp.ShapeError):
        gb.transfer_dictionary(src, (3, 4, 3), (10, 12, 4))


def test_live_install_other_k_and_transfer_between(cuda_device):
    img = inputs.synthetic_texture((16, 16), seed=1)
    mask = inputs.make_mask(img.shape, 0.4, "uniform-random", 1)
    cube = np.repeat(img[:, :, None], 3, axis=2) * np.array([1.0, 0.8, 0.6])
    cmask = inputs.make_mask(cube.shape, 0.4, "uniform-random", 2)
    with LiveProblem(img.shape, pp.PatchSpec((4, 4)), gb.Hyperparams(num_atoms=6), seed=1) as a, \
            LiveProblem(cube.shape, pp.PatchSpec((4, 4, 3)), gb.Hyperparams(num_atoms=10), seed=2) as b:
        a.submit_frame(img, mask)
        b.submit_frame(cube, cmask)
        _, _, sc_b = b.dictionary()
        atoms_a, pi_a, _ = a.dictionary()
        transfer_between(a, b)
        assert b.num_atoms == 6
        atoms_b, pi_b, sc_b2 = b.dictionary()
        want = gb.transfer_dictionary(gb.Dictionary(atoms_a.astype(np.float64), pi_a, (4, 4)), (4, 4, 3))
        assert np.abs(atoms_b - want.atoms).max() <= 1e-6 and np.array_equal(pi_b, pi_a)
        assert sc_b2.epoch == sc_b.epoch and sc_b2.gamma_eps == sc_b.gamma_eps   # precisions / epoch kept
        fr = b.submit_frame(cube, cmask)                    # sweeps with K = 6 now
        assert np.isfinite(fr.reconstruction).all()
        # an installed dictionary of yet another atom count
        rng = np.random.default_rng(3)
        d = gb.Dictionary(rng.standard_normal((9, 16)), rng.uniform(0.2, 0.8, 9), (4, 4))
        a.install_dictionary(d)
        assert a.num_atoms == 9
        assert np.isfinite(a.submit_frame(img, mask).reconstruction).all()
        with pytest.raises(ValueError):
            transfer_between(a, a)
        with pytest.raises(pp.ShapeError):
            transfer_between(b, a)
