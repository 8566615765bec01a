"""Keyed random streams: the draw contract shared with the reference.

Reference: pkg/src/patchbeam/rng.py:14-39.  Each stochastic site draws from a
numpy Philox4x64-10 stream keyed by (seed, domain, *subkeys).  In ``numpy``
RNG mode the host generates exactly these draws (bit-identical to the
reference's) and uploads them; in ``philox`` mode the device generates its own
counter-based Philox4x32-10 draws keyed by the same (seed, domain, epoch, atom,
patch) coordinates (statistically equivalent, not bit-identical).
"""

from __future__ import annotations

import numpy as np

DOMAIN_INIT = 1
DOMAIN_ATOM = 2
DOMAIN_CODE = 3
DOMAIN_PI = 4
DOMAIN_GAMMA = 5
DOMAIN_MASK = 6
DOMAIN_SYNTH = 7

_U32 = 0xFFFFFFFF
_U64 = 0xFFFFFFFFFFFFFFFF


def _seq(seed: int, *key: int) -> np.random.SeedSequence:
    return np.random.SeedSequence(entropy=int(seed) & _U64,
                                  spawn_key=tuple(int(k) & _U32 for k in key))


def keyed_rng(seed: int, *key: int) -> np.random.Generator:
    """Generator over the stream keyed by (seed, *key) — rng.py:25-32."""
    return np.random.Generator(np.random.Philox(_seq(seed, *key)))


def derive_seed(seed: int, *key: int) -> int:
    """rng.py:35-39."""
    return int(_seq(seed, *key).generate_state(1, dtype=np.uint64)[0])


def device_key(seed: int) -> tuple[int, int]:
    """64-bit Philox4x32 key for the device generator (philox mode)."""
    s = derive_seed(seed, 0x42323030)  # "B200"
    return s & _U32, (s >> 32) & _U32
