"""ORACLE — CPU restatement of the reference BPFA inpainting hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package, and only as the checker / CPU baseline — never as the thing
measured for the GPU arm, never on the product path.

Reference followed: /root/reference/pkg/src/patchbeam/{patches,bpfa,rng,_kernels}.py
(arXiv 2311.15061 "SenseAI", re-implemented there as the ``patchbeam`` package).

Parity pinning: the restatement is checked bit-for-bit (f64) against golden
fixtures produced by running the reference itself in the build container
(``tests/golden/make_golden.py``, committed with its outputs).
"""

from . import patches, bpfa, rng  # noqa: F401
