"""Accuracy/timing check of the compose seam (tensor-core path unless PB_COMPOSE_TC=0)."""
import sys, numpy as np, torch, ctypes, time
sys.path.insert(0, '.')
from paper_2311_15061_b200 import _lib
lib = _lib.load()
rng = np.random.default_rng(0)
for (n, p, k) in [(1000, 64, 64), (4097, 100, 256), (300, 16, 40), (2000, 256, 512), (1030225, 100, 256)]:
    ld = (n + 63) // 64 * 64
    z = (rng.random((k, ld)) < 0.5).astype(np.uint8)
    s = rng.standard_normal((k, ld)).astype(np.float32)
    d = rng.standard_normal((k, p)).astype(np.float32)
    zt, st, dt = (torch.from_numpy(x).cuda() for x in (z, s, d))
    out = torch.zeros((p, n), dtype=torch.float32, device='cuda')
    w = (z[:, :n] * s[:, :n]).astype(np.float64)
    ref = (d.astype(np.float64).T @ w) if n < 100000 else None
    # call through the seam: pb_compose_estimates(usage, weights, atoms, out, n, p, k, ld, accumulate, stream)
    st0 = torch.cuda.current_stream().cuda_stream
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(lib.pb_compose_estimates(zt.data_ptr(), st.data_ptr(), dt.data_ptr(), out.data_ptr(), n, p, k, ld, 0, st0))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        _lib.check(lib.pb_compose_estimates(zt.data_ptr(), st.data_ptr(), dt.data_ptr(), out.data_ptr(), n, p, k, ld, 0, st0))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    o = out.cpu().numpy().astype(np.float64)
    if ref is not None:
        err = np.abs(o - ref).max() / max(1e-30, np.abs(ref).max())
        print(f"n={n} p={p} k={k}: rel max err {err:.3e}  {ms:.3f} ms", flush=True)
    else:
        # spot check a few patches
        idx = rng.integers(0, n, 64)
        refs = d.astype(np.float64).T @ w[:, idx]
        err = np.abs(o[:, idx] - refs).max() / np.abs(refs).max()
        print(f"n={n} p={p} k={k}: spot rel max err {err:.3e}  {ms:.3f} ms", flush=True)
