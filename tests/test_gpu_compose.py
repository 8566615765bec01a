"""compose_estimates (bpfa.py:348-352, _kernels.py:133-145) on the tensor cores
(tcgen05.mma kind::tf32 with a 3xTF32 split, pb_compose_tc.cu) against an f64
NumPy reference: stated tolerance |err| <= 2e-5 * max|est| (3xTF32 keeps ~fp32
accuracy); tile tails (N % 128, P % 16, K % 32) and the accumulate mode
(tail averaging) included."""

import numpy as np
import pytest
import torch

from paper_2311_15061_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p,k", [(1, 1, 1), (127, 9, 7), (1000, 64, 64), (4097, 100, 256), (2000, 256, 40),
                                   (513, 36, 33)])
def test_compose_tensor_core_matches_f64(cuda_device, n, p, k):
    rng = np.random.default_rng(n + p + k)
    ld = (n + 63) // 64 * 64
    z = (rng.random((k, ld)) < 0.5).astype(np.uint8)
    s = rng.standard_normal((k, ld)).astype(np.float32)
    d = rng.standard_normal((k, p)).astype(np.float32)
    prev = rng.standard_normal((p, n)).astype(np.float32)
    ref = d.astype(np.float64).T @ (z[:, :n] * s[:, :n]).astype(np.float64)
    zt, st, dt = (torch.from_numpy(x).cuda() for x in (z, s, d))
    lib = _lib.load()
    for acc in (0, 1):
        out = torch.from_numpy(prev.copy()).cuda()
        _lib.check(lib.pb_compose_estimates(zt.data_ptr(), st.data_ptr(), dt.data_ptr(), out.data_ptr(), n, p, k, ld,
                                            acc, torch.cuda.current_stream().cuda_stream))
        want = ref + (prev.astype(np.float64) if acc else 0.0)
        got = out.cpu().numpy().astype(np.float64)
        assert np.abs(got - want).max() <= 2e-5 * max(1.0, np.abs(want).max()), (acc, np.abs(got - want).max())
