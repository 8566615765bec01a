"""Scratch: code-step time vs the narrow/wide split threshold (PB_CODE_SPLIT_AT)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_2311_15061_b200 import _lib  # noqa: E402
from paper_2311_15061_b200 import bpfa as gb  # noqa: E402
from paper_2311_15061_b200 import inputs  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402
from quick_timing_cfgs import CFGS  # noqa: E402

lib = _lib.load()
for cid in [int(a) for a in sys.argv[1].split(",")]:
    c = CFGS[cid]
    if len(c["shape"]) == 2:
        img = inputs.synthetic_texture(c["shape"], seed=0)
    else:
        base = inputs.synthetic_texture(c["shape"][:2], seed=0)
        spec = 0.5 + 0.5 * np.sin(np.linspace(0, 3 * np.pi, c["shape"][2]))
        img = base[:, :, None] * spec[None, None, :]
    mask = inputs.make_mask(c["shape"], c["ratio"], c["kind"], 0)
    pm = pp.extract_patches(img, mask, pp.PatchSpec(c["patch"]), len(c["shape"]) == 2)
    cnt = pm.observed_pn.sum(dim=0).cpu().numpy()
    if cnt is not None:
        qs = np.percentile(cnt, [50, 90, 99, 99.9, 100])
        print(f"cfg{cid}: count percentiles 50/90/99/99.9/max = {qs}")
    hp = gb.Hyperparams(num_atoms=c["k"])
    for t in sys.argv[2].split(","):
        if t == "auto":
            os.environ.pop("PB_CODE_SPLIT_AT", None)
        else:
            os.environ["PB_CODE_SPLIT_AT"] = t
        pm._cache.pop("ix_obs_version", None)  # rebuild the index with the new split
        gb.infer(pm, hp, 1, 0, rng="philox")
        torch.cuda.synchronize()
        lib.pb_phase_timing(1)
        gb.infer(pm, hp, 2, 0, rng="philox")
        torch.cuda.synchronize()
        ph = (ctypes.c_double * 4)(); ne = ctypes.c_int64()
        lib.pb_phase_read(ph, ctypes.byref(ne)); lib.pb_phase_timing(0)
        if cnt is not None and t != "auto":
            tt = int(t)
            frac = float((cnt > tt).mean()) if tt > 0 else 0.0
        else:
            frac = float("nan")
        ix = pm.index()
        print(f"  cfg{cid} split={t:>4} (index split {ix.split_count}, outliers {ix.n_outliers}) code {ph[2] / max(1, ne.value):.3f} ms/epoch  outlier frac {frac:.4f}", flush=True)
