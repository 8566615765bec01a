"""SADF dictionary files (formats.py:147-197) against files the reference wrote
(tests/golden/dict_*.sadf): byte-identical writer, identical reader, validation."""

import os

import numpy as np
import pytest

from paper_2311_15061_b200.bpfa import Dictionary
from paper_2311_15061_b200.formats import FormatError, read_dict, write_dict

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _src():
    z = np.load(os.path.join(GOLD, "dict_src.npz"))
    return Dictionary(z["atoms"], z["pi"], (3, 4))


def test_writer_is_byte_identical(tmp_path):
    d = _src()
    for name, pi in (("dict_k6_3x4.sadf", True), ("dict_k6_3x4_nopi.sadf", False)):
        out = tmp_path / name
        write_dict(out, d, include_pi=pi)
        assert out.read_bytes() == open(os.path.join(GOLD, name), "rb").read()


def test_reader_matches_reference_files():
    d = _src()
    r = read_dict(os.path.join(GOLD, "dict_k6_3x4.sadf"))
    assert r.patch_shape == (3, 4)
    assert np.array_equal(r.atoms, d.atoms.astype(np.float32).astype(np.float64))
    assert np.array_equal(r.pi, d.pi.astype(np.float32).astype(np.float64))
    r2 = read_dict(os.path.join(GOLD, "dict_k6_3x4_nopi.sadf"))
    assert np.array_equal(r2.pi, np.full(6, 0.5))


def test_reader_rejects_corruption(tmp_path):
    good = open(os.path.join(GOLD, "dict_k6_3x4.sadf"), "rb").read()
    bad = {"magic": b"XADF" + good[4:], "version": good[:4] + b"\x02" + good[5:], "truncated": good[:-3],
           "short_header": good[:10], "flags": good[:24] + b"\x02\x00\x00\x00" + good[28:]}
    for name, blob in bad.items():
        f = tmp_path / f"{name}.sadf"
        f.write_bytes(blob)
        with pytest.raises(FormatError):
            read_dict(f)
