"""In-kernel phase profile of the dictionary step (globaltimer), per BASELINE config."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_15061_b200 import _lib  # noqa: E402
from paper_2311_15061_b200 import bpfa as gb  # noqa: E402
from paper_2311_15061_b200 import inputs  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402
from tools.prof_epoch import CFGS  # noqa: E402

NAMES = ["pass start (acc, atoms)", "owner: partials copy wait", "elements (warp 0)", "pass-end CTA barrier",
         "owner: f64 reduce", "partials write", "grid sync 1", "owner phase", "grid sync 2", "delta load",
         "tile fill waits", "owner: draws + publish"]
for cid in [int(x) for x in sys.argv[1:]] or [3, 2]:
    c = CFGS[cid]
    img = inputs.synthetic_texture(c["shape"], seed=0) if len(c["shape"]) == 2 else \
        torch.rand(c["shape"], dtype=torch.float64).numpy()
    mask = inputs.make_mask(c["shape"], c["ratio"], c["kind"], 0)
    pm = pp.extract_patches(img, mask, pp.PatchSpec(c["patch"]), len(c["shape"]) == 2)
    hp = gb.Hyperparams(num_atoms=c["k"])
    st = gb.init_state(pm, hp, 0, "prior")
    gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
    lib = _lib.load()
    lib.pb_dict_profile(1, None)
    lib.pb_phase_timing(1)
    E = 3
    for _ in range(E):
        gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
    out = (ctypes.c_double * 12)()
    lib.pb_dict_profile(0, out)
    ph = (ctypes.c_double * 4)()
    ne = ctypes.c_int64()
    lib.pb_phase_read(ph, ctypes.byref(ne))
    print(f"cfg{cid}: N={pm.num_patches} nnz={pm.n_obs} dict {ph[1] / E:.3f} ms/epoch; in-kernel (thread 0, mean over CTAs, ms/epoch):")
    for nm, v in zip(NAMES, out):
        print(f"   {nm:20s} {v / 1e6 / E:8.3f}")
