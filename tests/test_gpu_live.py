"""The native live-frame path (pb_problem_submit_frame, host buffers) against
the Python API and the oracle.

* Cold frame (philox mode): the C++ problem and `bpfa.infer` + `reconstitute`
  consume identical device draws, so their reconstructions agree to f32 noise.
* Warm start across frames (pipeline.py:230-238): codes reset each frame, the
  dictionary / pi / gammas / epoch counter carry over; with data consistency the
  observed pixels are returned exactly.
* Reconstruction quality vs the oracle on the same frames (PSNR within 1.5 dB
  over a short live sequence: different random streams, same model; 1.5 dB).
"""

import ctypes

import numpy as np
import pytest

from paper_2311_15061_b200 import _lib
from paper_2311_15061_b200 import bpfa as gb
from paper_2311_15061_b200 import inputs
from paper_2311_15061_b200 import patches as pp
from paper_2311_15061_b200.metrics import psnr

pytestmark = pytest.mark.gpu


def _problem(shape, patch, k, epochs, warm, dc, seed=0):
    d = _lib.ProblemDesc()
    d.grid = pp.PatchSpec(patch).desc(shape)
    d.num_atoms = k
    for j, v in enumerate((1.0, 1.0, 1e-6, 1e-6, 1e-6, 1e-6)):
        d.hyper[j] = v
    d.seed = seed
    d.mean_subtract = 1
    d.epochs_per_frame = epochs
    d.warm_start = int(warm)
    d.data_consistency = int(dc)
    d.average_last = 1
    pr = ctypes.c_void_p()
    _lib.check(_lib.load().pb_problem_create(ctypes.byref(d), ctypes.byref(pr)))
    return pr


def _submit(pr, frame, mask):
    out = np.empty(frame.shape, dtype=np.float64)
    f = np.ascontiguousarray(frame, dtype=np.float64)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    _lib.check(_lib.load().pb_problem_submit_frame(pr, f.ctypes.data, m.ctypes.data, out.ctypes.data))
    return out


def test_native_cold_frame_matches_python_api(cuda_device):
    img = inputs.synthetic_texture((64, 72), seed=4)
    mask = inputs.make_mask(img.shape, 0.25, "uniform-random", 4)
    pr = _problem(img.shape, (8, 8), 16, 3, warm=False, dc=False, seed=9)
    try:
        native = _submit(pr, img, mask)
    finally:
        _lib.load().pb_problem_destroy(pr)
    pm = pp.extract_patches(img, mask, pp.PatchSpec((8, 8)), True)
    _, est = gb.infer(pm, gb.Hyperparams(num_atoms=16), 3, 9, rng="philox")
    py = pp.reconstitute(pm, est)
    assert np.abs(native - py).max() <= 1e-4


def test_native_warm_start_sequence(cuda_device):
    frames = inputs.synthetic_frames((64, 64), 4, seed=0)
    mask = inputs.make_mask((64, 64), 0.25, "line-hop", 0)
    pr = _problem((64, 64), (8, 8), 32, 2, warm=True, dc=True)
    lib = _lib.load()
    try:
        epochs = []
        for f in frames:
            out = _submit(pr, f, mask)
            assert np.array_equal(out[mask], f[mask])          # data consistency is exact
            s = _lib.Scalars()
            atoms = np.empty((32, 64), np.float32)
            pi = np.empty(32)
            _lib.check(lib.pb_problem_get_dictionary(pr, atoms.ctypes.data, pi.ctypes.data, ctypes.byref(s)))
            epochs.append(s.epoch)
            assert np.isfinite(atoms).all() and np.all((pi >= 0) & (pi <= 1))
        assert epochs == [2, 4, 6, 8]                           # the stream counter carries over
        assert lib.pb_problem_last_gpu_ms(pr) > 0
    finally:
        lib.pb_problem_destroy(pr)


def test_native_quality_tracks_oracle(cuda_device):
    from oracle import bpfa as ob
    from oracle import patches as op

    frames = inputs.synthetic_frames((48, 48), 3, seed=1)
    mask = inputs.make_mask((48, 48), 0.3, "uniform-random", 1)
    pr = _problem((48, 48), (6, 6), 12, 2, warm=True, dc=False)
    hp = ob.Hyper(num_atoms=12)
    st = None
    try:
        for f in frames:
            out = _submit(pr, f, mask)
            opm = op.extract_patches(f, mask, (6, 6), (), True)
            if st is not None:
                st.usage[:] = False
                st.weights[:] = 0.0
            st, est = ob.infer(opm, hp, 2, 0, state=st)
            ref = op.reconstitute(opm, est)
            assert abs(psnr(out, f) - psnr(ref, f)) <= 1.5, (psnr(out, f), psnr(ref, f))
    finally:
        _lib.load().pb_problem_destroy(pr)


def test_live_sequence_replay_matches_reference(golden, cuda_device):
    """The reference Pipeline's 3 warm-started frames (tests/golden/live.npz,
    produced by patchbeam itself) through this package's API in replay mode
    (the reference's own draw streams, same warm-start idiom): per-frame
    reconstruction within 1e-3 (f32 arithmetic; no Z flip expected) and PSNR
    within 0.05 dB."""
    g = golden("live.npz")
    hp = gb.Hyperparams(num_atoms=8)
    st = None
    for t in range(3):
        frame, mask = g[f"f{t}_frame"], g[f"f{t}_mask"]
        pm = pp.extract_patches(frame, mask, pp.PatchSpec((6, 6)), True)
        if st is not None:
            st.usage[:] = False
            st.weights[:] = 0.0
        st, est = gb.infer(pm, hp, 2, 0, rng="numpy", state=st)
        rec = pp.reconstitute(pm, est)
        ref = g[f"f{t}_recon"]
        assert abs(psnr(rec, frame) - psnr(ref, frame)) <= 0.05, t
        assert np.abs(rec - ref).max() <= 1e-3, (t, np.abs(rec - ref).max())


def test_native_replay_matches_reference_pipeline(golden, cuda_device):
    """The NATIVE live path (pb_problem_submit_frame, host buffers) in replay
    mode against the reference Pipeline's 3 warm-started frames
    (tests/golden/live.npz: Pipeline defaults — init "data", 2 epochs/frame,
    DC off): per-frame reconstruction within 1e-3 and PSNR within 0.05 dB."""
    from paper_2311_15061_b200.live import LiveProblem

    g = golden("live.npz")
    shape = g["f0_frame"].shape
    with LiveProblem(shape, pp.PatchSpec((6, 6)), gb.Hyperparams(num_atoms=8), seed=0, epochs_per_frame=2,
                     rng="numpy") as lp:
        for t in range(3):
            frame, mask = g[f"f{t}_frame"], g[f"f{t}_mask"]
            rec = lp.submit_frame(frame, mask).reconstruction
            ref = g[f"f{t}_recon"]
            assert abs(psnr(rec, frame) - psnr(ref, frame)) <= 0.05, t
            assert np.abs(rec - ref).max() <= 1e-3, (t, np.abs(rec - ref).max())
            atoms, _, sc = lp.dictionary()
            assert np.abs(atoms - g[f"f{t}_atoms"]).max() <= 1e-4
            assert sc.epoch == 2 * (t + 1)


def test_native_frozen_data_init_matches_oracle(cuda_device):
    """freeze_dict without an installed dictionary: the native cold
    start seeds the atoms from the K patches with the most observed elements
    (bpfa.py:126-134, on device) and keeps them; replay mode then reproduces the
    oracle's frozen inference."""
    from oracle import bpfa as ob
    from oracle import patches as op
    from paper_2311_15061_b200.live import LiveProblem

    img = inputs.synthetic_texture((40, 44), seed=3)
    mask = inputs.make_mask(img.shape, 0.3, "uniform-random", 3)
    k = 10
    opm = op.extract_patches(img, mask, (6, 6), (), True)
    hp = ob.Hyper(num_atoms=k)
    ost = ob.init_state(opm, hp, 5, "data")
    want_atoms = ost.atoms.copy()
    ost, oest = ob.infer(opm, hp, 3, 5, freeze_dict=True, state=ost)
    orec = op.reconstitute(opm, oest)
    for rng in ("numpy", "philox"):
        with LiveProblem(img.shape, pp.PatchSpec((6, 6)), gb.Hyperparams(num_atoms=k), seed=5, epochs_per_frame=3,
                         freeze_dict=True, rng=rng) as lp:
            rec = lp.submit_frame(img, mask).reconstruction
            atoms, _, _ = lp.dictionary()
        assert np.abs(atoms - want_atoms).max() <= 1e-6, rng   # data-seeded and frozen
        if rng == "numpy":
            assert np.abs(rec - orec).max() <= 1e-3


def test_cached_mask_frame_refresh_bit_identical_to_extraction(cuda_device):
    """A cached mask sends a 2-D frame's observed values straight from the frame
    into the compact index order (k_refresh_frame2d) instead of the dense
    extraction + value refresh: the same bits.  Problem A keeps one mask (fused
    refresh from its second frame on); problem B re-draws the same mask before
    every frame (pure-explore adaptive mask at a fixed frame index), which
    invalidates its index, so B always extracts densely."""
    from paper_2311_15061_b200.live import LiveProblem

    frames = inputs.synthetic_frames((72, 80), 4, seed=2)
    hp = gb.Hyperparams(num_atoms=16)
    with LiveProblem((72, 80), pp.PatchSpec((8, 8)), hp, seed=4, epochs_per_frame=2) as a, \
            LiveProblem((72, 80), pp.PatchSpec((8, 8)), hp, seed=4, epochs_per_frame=2) as b:
        mask = b.adaptive_mask(0.3, 0.0, seed=1, frame_index=0)
        for f in frames:
            assert np.array_equal(b.adaptive_mask(0.3, 0.0, seed=1, frame_index=0), mask)
            ra = a.submit_frame(f, mask).reconstruction
            rb = b.submit_frame(f, mask).reconstruction
            assert np.array_equal(ra, rb)
