"""Device-resident live tail against the oracle restatement
(oracle/sampling.py, pinned to the reference by tests/golden/live_tail.npz):

* uint8 wire panels: bit-exact with round(clip(x,0,1)*255) of the returned
  reconstruction / of frame*mask (rank 2 and slice 0 of rank 3);
* residual map: bit-exact (recon_t - recon_{t-1})^2, zeros on the first frame;
* adaptive sampler: budget exact; exploit set bit-exact with the reference's
  stable argsort (with exploit_fraction = 1 the mask equals the reference's
  mask); the explore part is a device stream — checked for disjointness,
  count and uniformity (each candidate's hit rate within 5 sigma);
* errors: negative residuals and non-2D/3D panels refuse.
"""

import numpy as np
import pytest

from oracle import sampling as osm
from paper_2311_15061_b200 import _lib
from paper_2311_15061_b200 import inputs
from paper_2311_15061_b200.bpfa import Hyperparams
from paper_2311_15061_b200.live import LiveProblem, adaptive_mask
from paper_2311_15061_b200.patches import PatchSpec, ShapeError

pytestmark = pytest.mark.gpu


def test_panels_and_residual_map(cuda_device):
    frames = inputs.synthetic_frames((24, 24), 3, seed=0)
    mask = inputs.make_mask((24, 24), 0.3, "uniform-random", 0)
    with LiveProblem((24, 24), PatchSpec((6, 6)), Hyperparams(num_atoms=8), epochs_per_frame=2) as lp:
        prev = None
        for f in frames:
            fr = lp.submit_frame(f, mask, panels=True)
            assert np.array_equal(fr.panel, osm.quantize_panel(fr.reconstruction))
            assert np.array_equal(fr.masked_panel, osm.quantize_panel(f * mask))
            assert np.array_equal(lp.residual_map(), osm.residual_map(fr.reconstruction, prev))
            prev = fr.reconstruction
            assert fr.gpu_ms > 0


def test_data_consistency_and_rank3_panel(cuda_device):
    rng = np.random.default_rng(3)
    cube = rng.random((12, 10, 3))
    mask = rng.random(cube.shape) < 0.4
    with LiveProblem(cube.shape, PatchSpec((4, 4, 3)), Hyperparams(num_atoms=6), data_consistency=True) as lp:
        fr = lp.submit_frame(cube, mask, panels=True)
        assert np.array_equal(fr.reconstruction[mask], cube[mask])
        assert fr.panel.shape == (12, 10)
        assert np.array_equal(fr.panel, osm.quantize_panel(fr.reconstruction))
    with LiveProblem((40,), PatchSpec((5,)), Hyperparams(num_atoms=4)) as lp:
        with pytest.raises(ValueError):
            lp.submit_frame(np.zeros(40), np.ones(40, bool), panels=True)


@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_adaptive_exploit_matches_reference(golden, cuda_device, case):
    g = golden("live_tail.npz")
    ratio, ef, seed, fi = g[f"a{case}_spec"]
    res, ref_mask = g[f"a{case}_res"], g[f"a{case}_mask"]
    mask, all_zero = adaptive_mask(res, ratio, ef, int(seed), int(fi))
    budget, n_exploit = osm.adaptive_split(ratio, ef, res.size)
    assert not all_zero and mask.sum() == budget == ref_mask.sum()
    ex = osm.adaptive_exploit(res, ratio, ef)
    assert mask.ravel()[ex].all()
    if n_exploit == budget:            # pure exploit: the whole mask is reference-exact
        assert np.array_equal(mask, ref_mask)


def test_adaptive_explore_is_uniform_and_keyed(cuda_device):
    rng = np.random.default_rng(11)
    res = rng.random((20, 20)) * (rng.random((20, 20)) < 0.5)
    ex = set(osm.adaptive_exploit(res, 0.2, 0.5).tolist())
    budget, n_exploit = osm.adaptive_split(0.2, 0.5, res.size)
    hits = np.zeros(res.size)
    trials = 300
    for t in range(trials):
        m, _ = adaptive_mask(res, 0.2, 0.5, seed=7, frame_index=t)
        flat = np.flatnonzero(m.ravel())
        assert len(flat) == budget and ex <= set(flat.tolist())
        hits[flat] += 1
    free = np.array([i for i in range(res.size) if i not in ex])
    p = (budget - n_exploit) / len(free)
    rate = hits[free] / trials
    assert np.all(np.abs(rate - p) <= 5 * np.sqrt(p * (1 - p) / trials))
    a, _ = adaptive_mask(res, 0.2, 0.5, seed=7, frame_index=3)
    b, _ = adaptive_mask(res, 0.2, 0.5, seed=7, frame_index=3)
    c, _ = adaptive_mask(res, 0.2, 0.5, seed=8, frame_index=3)
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_adaptive_zero_and_invalid(cuda_device):
    m, all_zero = adaptive_mask(np.zeros((16, 16)), 0.25, 0.5, seed=1)
    assert all_zero and m.sum() == osm.sample_budget(0.25, 256)
    with pytest.raises(ValueError):
        adaptive_mask(-np.ones((4, 4)), 0.25)
    with pytest.raises(ValueError):
        adaptive_mask(np.ones((4, 4)), 1.5)


def test_problem_adaptive_loop(cuda_device):
    """Frame t's mask comes from frame t-1's residual map, on device."""
    frames = inputs.synthetic_frames((32, 32), 4, seed=2)
    with LiveProblem((32, 32), PatchSpec((6, 6)), Hyperparams(num_atoms=8)) as lp:
        mask = lp.adaptive_mask(0.3, 0.5, seed=0)           # no residual yet: uniform
        assert mask.sum() == osm.sample_budget(0.3, 1024)
        for f in frames:
            lp.submit_frame(f, mask)
            res = lp.residual_map()
            nxt = lp.adaptive_mask(0.3, 0.5, seed=0)
            if res.any():
                assert nxt.ravel()[osm.adaptive_exploit(res, 0.3, 0.5)].all()
            mask = nxt


def test_install_dictionary_pending_and_live(cuda_device, tmp_path):
    """Pipeline._install_dictionary semantics (pipeline.py:145-167) through a
    SADF round trip: pending before the first frame (frozen: the sweep keeps it
    bit-exact), and a live replacement keeps the epoch counter."""
    from paper_2311_15061_b200.bpfa import Dictionary
    from paper_2311_15061_b200.formats import read_dict, write_dict

    rng = np.random.default_rng(4)
    d = Dictionary(rng.standard_normal((8, 36)).astype(np.float32).astype(np.float64), rng.uniform(0.1, 0.9, 8),
                   (6, 6))
    write_dict(tmp_path / "d.sadf", d)
    d = read_dict(tmp_path / "d.sadf")
    frames = inputs.synthetic_frames((24, 24), 2, seed=1)
    mask = inputs.make_mask((24, 24), 0.3, "uniform-random", 1)
    with LiveProblem((24, 24), PatchSpec((6, 6)), Hyperparams(num_atoms=8), epochs_per_frame=2) as lp:
        lp.install_dictionary(d, freeze=True)                  # pending: seeds the cold start
        lp.submit_frame(frames[0], mask)
        atoms, pi, sc = lp.dictionary()
        assert np.array_equal(atoms, d.atoms.astype(np.float32)) and sc.epoch == 2
        lp.install_dictionary(lp.snapshot_dictionary(), freeze=False)   # live: epoch carries over
        lp.submit_frame(frames[1], mask)
        atoms2, _, sc2 = lp.dictionary()
        assert sc2.epoch == 4 and not np.array_equal(atoms2, atoms)
        lp.install_dictionary(Dictionary(np.zeros((5, 36)), np.full(5, 0.5), (6, 6)))   # another K: re-sized
        assert lp.num_atoms == 5 and lp.dictionary()[0].shape == (5, 36)
        with pytest.raises(ShapeError):
            lp.install_dictionary(Dictionary(np.zeros((5, 25)), np.full(5, 0.5), (5, 5)))


def test_atlas_on_device_matches_reference(golden, cuda_device):
    """server.render_dictionary_atlas (server.py:84-120) on device vs the
    reference's own canvases (f32-exact atoms): bit-exact f64, exact uint8."""
    from paper_2311_15061_b200.bpfa import Dictionary
    from paper_2311_15061_b200.display import pack_wireframe, render_dictionary_atlas, unpack_wireframe

    g = golden("atlas.npz")
    for name in ("a2", "a3", "a1", "a2sq"):
        d = Dictionary(g[f"{name}_atoms"], g[f"{name}_pi"], tuple(int(b) for b in g[f"{name}_shape"]))
        c = render_dictionary_atlas(d)
        assert np.array_equal(c, g[f"{name}_canvas"]), name
        u8 = render_dictionary_atlas(d, as_uint8=True)
        assert np.array_equal(u8, osm.quantize_panel(g[f"{name}_canvas"])), name
        hdr, back = unpack_wireframe(pack_wireframe(2, 7, 3, u8))
        assert np.array_equal(back, u8) and hdr["problem_id"] == 7 and hdr["frame_id"] == 3
    with pytest.raises(ValueError):
        render_dictionary_atlas(Dictionary(np.zeros((2, 16)), np.zeros(2), (2, 2, 2, 2)))
    with LiveProblem((24, 24), PatchSpec((6, 6)), Hyperparams(num_atoms=8)) as lp:
        lp.submit_frame(inputs.synthetic_frames((24, 24), 1, seed=0)[0], np.ones((24, 24), bool))
        atoms, pi, _ = lp.dictionary()
        assert np.array_equal(lp.render_atlas(), osm.quantize_panel(osm.render_dictionary_atlas(atoms, pi, (6, 6))))


@pytest.mark.parametrize("shape,levels,ratio", [((1, 1), 3, 1.0), ((33, 47), 4, 0.3), ((512, 512), 7, 0.25),
                                                ((1000, 1100), 1000, 0.1), ((640, 480), 2, 0.5),
                                                ((257, 129), 5, 1.0), ((3000, 3000), 50, 0.0005)])
def test_adaptive_exploit_select_ties_exact(cuda_device, shape, levels, ratio):
    """Pure exploit on residuals with heavy ties (few distinct levels, zeros,
    -0.0): the device radix select (pb_select.cu) takes exactly the first
    n_exploit of the reference's argsort(-r, kind="stable") — every key above
    the threshold and the lowest-index ties at it."""
    rng = np.random.default_rng(levels)
    res = rng.integers(0, levels, size=shape).astype(np.float64) * 0.37
    res[rng.random(shape) < 0.05] = -0.0
    if res.max() == 0:
        res.flat[0] = 1.0
    mask, all_zero = adaptive_mask(res, ratio, 1.0, 0, 0)
    budget, n_exploit = osm.adaptive_split(ratio, 1.0, res.size)
    want = np.zeros(res.size, bool)
    want[np.argsort(-res.ravel(), kind="stable")[:n_exploit]] = True
    assert not all_zero and n_exploit == budget
    assert np.array_equal(mask.ravel(), want)
