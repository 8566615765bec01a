"""ORACLE (test infrastructure only): keyed counter-based random streams.

Restates reference pkg/src/patchbeam/rng.py:14-39 — one numpy Philox4x64-10
stream per (seed, domain, *subkeys); subkeys folded to uint32, the seed is the
64-bit SeedSequence entropy root.
"""

from __future__ import annotations

import numpy as np

# rng.py:14-20
DOMAIN_INIT = 1
DOMAIN_ATOM = 2
DOMAIN_CODE = 3
DOMAIN_PI = 4
DOMAIN_GAMMA = 5
DOMAIN_MASK = 6
DOMAIN_SYNTH = 7

_U32 = 0xFFFFFFFF
_U64 = 0xFFFFFFFFFFFFFFFF


def keyed_rng(seed: int, *key: int) -> np.random.Generator:
    """rng.py:25-32."""
    parts = tuple(int(k) & _U32 for k in key)
    ss = np.random.SeedSequence(entropy=int(seed) & _U64, spawn_key=parts)
    return np.random.Generator(np.random.Philox(ss))
