"""Profiling driver: one warm-up epoch then `epochs` epochs of one BASELINE config
(philox mode).  Used under ncu: the sweep kernels of epoch 2+ are the captures."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_15061_b200 import bpfa as gb  # noqa: E402
from paper_2311_15061_b200 import inputs  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402

CFGS = {
    1: dict(shape=(256, 256), ratio=0.25, kind="uniform-random", patch=(8, 8), k=64),
    2: dict(shape=(1024, 1024), ratio=0.10, kind="uniform-random", patch=(10, 10), k=256),
    3: dict(shape=(512, 512), ratio=0.25, kind="line-hop", patch=(8, 8), k=256),
    4: dict(shape=(256, 256, 128), ratio=0.20, kind="uniform-random", patch=(8, 8, 4), k=512),
    5: dict(shape=(4096, 4096), ratio=0.10, kind="uniform-random", patch=(8, 8), k=256),
}
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = CFGS[cid]
rng = torch.Generator().manual_seed(0)
img = torch.rand(c["shape"], generator=rng, dtype=torch.float64).numpy() if len(c["shape"]) > 2 \
    else inputs.synthetic_texture(c["shape"], seed=0)
mask = inputs.make_mask(c["shape"], c["ratio"], c["kind"], 0)
pm = pp.extract_patches(img, mask, pp.PatchSpec(c["patch"]), len(c["shape"]) == 2)
hp = gb.Hyperparams(num_atoms=c["k"])
st = gb.init_state(pm, hp, 0, "prior")
gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
torch.cuda.synchronize()
for _ in range(epochs):
    gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
torch.cuda.synchronize()
print("ok", pm.num_patches, pm.n_obs)
