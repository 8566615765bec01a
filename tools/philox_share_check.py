"""Bit-identity check for library variants on the Philox path: a crop of the
configs[3] cube (multi-lane code-step patches) through 3 sweeps from the same
seed; prints a hash of Z, S and D.  python tools/philox_share_check.py
[PB200_LIB_VARIANT=name]."""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_15061_b200 import bpfa as gb  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402

cfg = dict(bench.CFGS[3])
img, mask = bench.config_inputs(cfg)
img, mask = np.ascontiguousarray(img[:48, :48]), np.ascontiguousarray(mask[:48, :48])
pm = pp.extract_patches(img, mask, pp.PatchSpec(cfg["patch"]), False)
hp = gb.Hyperparams(num_atoms=cfg["k"])
st = gb.init_state(pm, hp, 5, "prior")
for _ in range(3):
    gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
torch.cuda.synchronize()
h = st.to_host()
d = hashlib.sha256()
for key in ("usage", "weights"):
    d.update(np.ascontiguousarray(h[key]).tobytes())
d.update(np.ascontiguousarray(st.dictionary.atoms.cpu().numpy()).tobytes())
print("N", pm.num_patches, "cmax", int(pm.counts.max()), "hash", d.hexdigest()[:16])
