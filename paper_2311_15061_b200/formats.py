"""Dictionary files (SADF) for --dict-in/--dict-out and dictionary transfer
between problems (formats.py:19-31, 147-204 of the reference): little-endian,
float32 payload, every header field and the exact payload length validated.
Host I/O — the dictionary then goes to the device through
``LiveProblem.install_dictionary`` / ``bpfa.install_dictionary``.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .bpfa import Dictionary

DICT_MAGIC = b"SADF"
FORMAT_VERSION = 1
FLAG_PI = 0x1
MAX_RANK = 4
_MAX_DIM = 1 << 24
_MAX_ATOMS = 1 << 20


class FormatError(ValueError):
    """Malformed, truncated or unsupported file content (formats.py:30-31)."""


def _unpack(data: bytes, pos: int, fmt: str):
    size = struct.calcsize(fmt)
    if pos + size > len(data):
        raise FormatError("truncated file header")
    return struct.unpack_from(fmt, data, pos)


def write_dict(path, dictionary: Dictionary, include_pi: bool = True) -> None:
    """formats.py:147-161: magic, (version, K, rank), patch shape, flags, atoms
    (K, P) f32, then pi (K) f32 when flagged."""
    d = dictionary.to_host() if hasattr(dictionary, "to_host") else dictionary
    atoms = np.ascontiguousarray(np.asarray(d.atoms), dtype="<f4")
    shape = tuple(int(b) for b in d.patch_shape)
    k = atoms.shape[0]
    blob = (DICT_MAGIC + struct.pack("<III", FORMAT_VERSION, k, len(shape)) + struct.pack(f"<{len(shape)}I", *shape)
            + struct.pack("<I", FLAG_PI if include_pi else 0) + atoms.tobytes())
    if include_pi:
        blob += np.ascontiguousarray(np.asarray(d.pi), dtype="<f4").tobytes()
    Path(path).write_bytes(blob)


def read_dict(path) -> Dictionary:
    """formats.py:164-197 (atoms and pi widened to f64; pi = 0.5 when absent)."""
    data = Path(path).read_bytes()
    if data[:4] != DICT_MAGIC:
        raise FormatError("bad dictionary file magic")
    version, k, ndims = _unpack(data, 4, "<III")
    pos = 16
    if version != FORMAT_VERSION:
        raise FormatError(f"unsupported dictionary file version {version}")
    if not 1 <= k <= _MAX_ATOMS:
        raise FormatError(f"invalid atom count {k}")
    if not 1 <= ndims <= MAX_RANK:
        raise FormatError(f"invalid patch rank {ndims}")
    shape = _unpack(data, pos, f"<{ndims}I")
    pos += 4 * ndims
    if any(b < 1 or b > _MAX_DIM for b in shape):
        raise FormatError(f"invalid patch shape {shape}")
    (flags,) = _unpack(data, pos, "<I")
    pos += 4
    if flags & ~FLAG_PI:
        raise FormatError(f"unknown dictionary flags 0x{flags:x}")
    p = int(np.prod(shape))
    expected = k * p * 4 + (k * 4 if flags & FLAG_PI else 0)
    payload = data[pos:]
    if len(payload) != expected:
        raise FormatError(f"dictionary payload is {len(payload)} bytes, expected {expected}")
    atoms = np.frombuffer(payload[:k * p * 4], dtype="<f4").reshape(k, p).astype(np.float64)
    pi = (np.frombuffer(payload[k * p * 4:], dtype="<f4").astype(np.float64) if flags & FLAG_PI
          else np.full(k, 0.5, dtype=np.float64))
    return Dictionary(atoms=atoms, pi=pi, patch_shape=tuple(int(b) for b in shape))
