"""CPU-side checks of the C ABI boundary and host logic (no GPU needed).

* libpb200.so loads and exports exactly the functions include/pb200.h declares;
* the ctypes struct layouts match the C structs;
* pb_grid_counts (pure host logic) matches the reference grid formula and its
  ShapeError cases (patches.py:54-70) and a brute-force count (oracles.py:176-186).
"""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2311_15061_b200 import _lib
from paper_2311_15061_b200.patches import PatchSpec, ShapeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "pb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = _header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), "ctypes signatures out of sync with pb200.h"
    assert lib.pb_version() >= 1


def test_struct_layouts():
    assert ctypes.sizeof(_lib.Scalars) == 40
    assert ctypes.sizeof(_lib.GridDesc) == 4 + 4 + 8 * 4 + 4 * 4 + 4 * 4  # incl. padding after rank
    assert _lib.EpochDesc.values.offset % 8 == 0


def _brute(shape, patch, stride):
    c = 1
    for m, b, s in zip(shape, patch, stride):
        k, o = 0, 0
        while o + b <= m:
            k += 1
            o += s
        c *= k
    return c


def test_grid_counts_host_and_abi_agree_with_brute_force():
    rng = np.random.default_rng(4)
    lib = _lib.load()
    for ndim in (1, 2, 3, 4):
        for _ in range(12):
            shape = tuple(int(rng.integers(1, 9)) for _ in range(ndim))
            patch = tuple(int(rng.integers(1, m + 1)) for m in shape)
            stride = tuple(int(rng.integers(1, 4)) for _ in range(ndim))
            spec = PatchSpec(patch, stride)
            want = _brute(shape, patch, stride)
            assert spec.num_patches(shape) == want
            counts = (ctypes.c_int64 * 4)()
            n = ctypes.c_int64()
            p = ctypes.c_int32()
            assert lib.pb_grid_counts(ctypes.byref(spec.desc(shape)), counts, ctypes.byref(n), ctypes.byref(p)) == 0
            assert n.value == want and p.value == int(np.prod(patch))
            assert tuple(counts[:ndim]) == spec.grid_counts(shape)


def test_grid_shape_errors_map_to_shape_error():
    lib = _lib.load()
    spec = PatchSpec((5, 2))
    with pytest.raises(ShapeError):
        spec.grid_counts((4, 4))
    g = spec.desc((4, 4))
    assert lib.pb_grid_counts(ctypes.byref(g), None, None, None) == _lib.PB_ESHAPE
    assert b"exceeds" in lib.pb_last_error()
    with pytest.raises(ShapeError):
        PatchSpec((2, 2), (1,))
    with pytest.raises(ShapeError):
        PatchSpec((0, 2))
    with pytest.raises(ShapeError):
        PatchSpec((2,)).grid_counts((3, 3))
    with pytest.raises(ShapeError):
        PatchSpec((1, 1, 1, 1, 1)).grid_counts((2, 2, 2, 2, 2))


def test_spanning_dimension_single_position_any_stride():
    for stride in (1, 2, 5):
        assert PatchSpec((3, 4), (1, stride)).grid_counts((6, 4))[1] == 1


def test_hyperparams_validation():
    from paper_2311_15061_b200.bpfa import Hyperparams

    with pytest.raises(ValueError):
        Hyperparams(num_atoms=0)
    with pytest.raises(ValueError):
        Hyperparams(noise_rate=0.0)
    assert Hyperparams().as6() == (1.0, 1.0, 1e-6, 1e-6, 1e-6, 1e-6)
