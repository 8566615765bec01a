"""Scratch timing of the device path on the BASELINE configs (not the bench)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_2311_15061_b200 import bpfa as gb  # noqa: E402
from paper_2311_15061_b200 import inputs  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402

from quick_timing_cfgs import CFGS  # noqa: E402

for cid in [int(a) for a in sys.argv[1:]] or [1, 3, 2]:
    c = CFGS[cid]
    if len(c["shape"]) == 2:
        img = inputs.synthetic_texture(c["shape"], seed=0)
    else:  # hyperspectral-like cube: per-band texture with a smooth spectral modulation
        base = inputs.synthetic_texture(c["shape"][:2], seed=0)
        spec = 0.5 + 0.5 * np.sin(np.linspace(0, 3 * np.pi, c["shape"][2]))
        img = base[:, :, None] * spec[None, None, :]
    mask = inputs.make_mask(c["shape"], c["ratio"], c["kind"], 0)
    pm = pp.extract_patches(img, mask, pp.PatchSpec(c["patch"]), len(c["shape"]) == 2)
    hp = gb.Hyperparams(num_atoms=c["k"])
    st, est = gb.infer(pm, hp, 1, 0, rng="philox")  # warm-up
    torch.cuda.synchronize()
    import ctypes
    from paper_2311_15061_b200 import _lib
    lib = _lib.load()
    lib.pb_phase_timing(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st, est = gb.infer(pm, hp, c["epochs"], 0, rng="philox")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ph = (ctypes.c_double * 4)(); ne = ctypes.c_int64()
    lib.pb_phase_read(ph, ctypes.byref(ne)); lib.pb_phase_timing(0)
    print("  phases ms/epoch [resid, dict, code, stats]:", [round(ph[i] / max(1, ne.value), 3) for i in range(4)])
    rec = pp.reconstitute(pm, est, dc_original=img, dc_mask=mask)
    from paper_2311_15061_b200.metrics import psnr
    upd = pm.num_patches * c["k"] * c["epochs"]
    print(f"cfg{cid}: N={pm.num_patches} K={c['k']} epochs={c['epochs']} {ms:.2f} ms "
          f"({ms / c['epochs']:.3f} ms/epoch) {upd / ms * 1e3:.3e} upd/s psnr={psnr(rec, img):.2f}", flush=True)
