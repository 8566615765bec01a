"""Steady-state device sweep timing of BASELINE configs (scratch A/B tool):
python tools/sweep_timing.py [cfg ids...] [--steps N]; PB200_LIB_VARIANT=name picks
a library variant.  Prints ms per sweep and the dictionary / code phases."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_15061_b200 import _lib  # noqa: E402
from paper_2311_15061_b200 import bpfa as gb  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 5
if "--steps" in sys.argv:
    args.remove(str(steps))
split = int(sys.argv[sys.argv.index("--split") + 1]) if "--split" in sys.argv else 0
if "--split" in sys.argv:
    args.remove(str(split))
lib = _lib.load()
for cid in [int(a) for a in args] or [1]:
    cfg = bench.CFGS[cid]
    img, mask = bench.config_inputs(cfg)
    pm = pp.extract_patches(img, mask, pp.PatchSpec(cfg["patch"]), len(cfg["shape"]) == 2)
    pm.split_request = split
    ix = pm.index()
    hp = gb.Hyperparams(num_atoms=cfg["k"])
    st = gb.init_state(pm, hp, 0, "prior")
    for _ in range(3):
        gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
    torch.cuda.synchronize()
    lib.pb_phase_timing(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ph = (ctypes.c_double * 4)()
    ne = ctypes.c_int64()
    lib.pb_phase_read(ph, ctypes.byref(ne))
    lib.pb_phase_timing(0)
    n = max(1, ne.value)
    print(f"cfg{cid} {_lib.LIB_PATH.split('/')[-1]}: {ms:.3f} ms/sweep  dict {ph[1] / n:.3f}  code {ph[2] / n:.3f}  "
          f"{pm.num_patches * cfg['k'] / ms / 1e6:.2f} G upd/s  split {ix.split_count} (cmax {ix.cmax}, "
          f"{ix.n_outliers} wide)", flush=True)
    del st, pm
    torch.cuda.empty_cache()
