"""Replay parity at BASELINE sizes (VERDICT r01 "pin parity at
BASELINE scale").

Teacher-forced replay (tests/_parity.py): each epoch starts from the reference
state, both sides consume the reference's own draw streams, and the device epoch
must match the reference epoch within the stated tolerances of tests/_parity.py
(S <= 1e-5 rel, D <= 1e-5 abs, pi / gamma_s <= 1e-6 rel, gamma_eps <= 1e-4 rel,
Z flips <= max(2, 1e-6 N K)).  The reference epochs are produced on the box by
the oracle, which is bit-exact to patchbeam (tests/test_oracle_golden.py).

* configs[0] in full: 256x256 STEM-like, 25 % uniform, 8x8, K = 64, all 10 epochs;
* configs[2]: one 512x512 line-hop 25 % frame, 8x8, K = 256, both epochs of a
  frame (the first from Z = 0, the second through the full dictionary step);
* configs[1] band: 160 rows of the 1024x1024 10 % frame, 10x10, K = 256
  (153,265 patches >= 2^17: the warp-claimed code step with pitch-8 windows
  that configs[1] runs), 2 epochs;
* configs[3] crop: a 24x24x16 crop of the cube, 8x8x4, K = 64 (multi-lane code
  step, 16-warp dictionary variant), 3 epochs;
* configs[4] band: 40 rows of the 4096x4096 10 % frame, 8x8, K = 256 (135K
  patches, the full row width), 2 epochs;
* cube with a dictionary larger than shared memory: 8x8x4 patches (P = 256),
  K = 160 > the ~100 atoms a code-step chunk holds, ~64 observed per patch (the
  2- and 4-lane variants restaging every chunk per block of patches, as
  configs[3] with K = 512 does), 2 epochs.
"""

import numpy as np
import pytest

from _parity import check, fmt, teacher_forced
from paper_2311_15061_b200 import inputs

pytestmark = pytest.mark.gpu


def _run(name, img, mask, patch, k, epochs, seed=0, **kw):
    stats, (pm, _, _) = teacher_forced(img, mask, patch, k, epochs, seed, **kw)
    n = pm.num_patches
    for s in stats:
        print(name, fmt(s))
    for s in stats:
        check(s, n, k, f"{name}/e{s['epoch']}")
    return stats


def test_configs0_full_teacher_forced():
    img = inputs.stem_lattice((256, 256), seed=0)
    mask = inputs.make_mask((256, 256), 0.25, "uniform-random", 0)
    _run("cfg0", img, mask, (8, 8), 64, 10)


def test_configs2_frame_teacher_forced():
    frame = inputs.synthetic_frames((512, 512), 1, seed=0)[0]
    mask = inputs.make_mask((512, 512), 0.25, "line-hop", 0)
    _run("cfg2", frame, mask, (8, 8), 256, 2)


def test_configs1_band_teacher_forced():
    img = inputs.stem_lattice((1024, 1024), seed=0)[:160]
    mask = inputs.make_mask((1024, 1024), 0.10, "uniform-random", 0)[:160]
    stats = _run("cfg1band", np.ascontiguousarray(img), np.ascontiguousarray(mask), (10, 10), 256, 2)
    assert len(stats) == 2


def test_configs3_crop_teacher_forced():
    base = inputs.stem_lattice((24, 24), seed=0)
    spec = 0.5 + 0.5 * np.sin(np.linspace(0.0, 3.0 * np.pi, 16))
    img = base[:, :, None] * spec[None, None, :]
    mask = inputs.make_mask(img.shape, 0.20, "uniform-random", 0)
    _run("cfg3crop", img, mask, (8, 8, 4), 64, 3, mean_subtract=False)


def test_configs4_band_teacher_forced():
    img = inputs.stem_lattice((4096, 4096), seed=0)[:40]
    mask = inputs.make_mask((4096, 4096), 0.10, "uniform-random", 0)[:40]
    _run("cfg4band", np.ascontiguousarray(img), np.ascontiguousarray(mask), (8, 8), 256, 2)


def test_cube_chunked_dictionary_teacher_forced():
    rng = np.random.default_rng(7)
    base = inputs.stem_lattice((20, 22), seed=1)
    img = base[:, :, None] * (0.6 + 0.4 * rng.random(12))[None, None, :]
    mask = inputs.make_mask(img.shape, 0.25, "uniform-random", 1)
    _run("cubechunk", img, mask, (8, 8, 4), 160, 2, mean_subtract=False)
