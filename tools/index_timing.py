"""Time the observed-element index build (extract + pb_build_index) at configs[1]/[2]/[4] sizes."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402

for cfg in (bench.CFG, bench.LIVE, bench.OTHER_CFGS[4]):
    img, mask = bench.config_inputs(cfg) if "what" in cfg else bench.workload_inputs(cfg)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pm = pp.extract_patches(img, mask, pp.PatchSpec(cfg["patch"]), True)
        pm.index()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    print(f"{cfg['shape']} {cfg['patch']}: extract + index {1e3 * (t1 - t0):.2f} ms (N={pm.num_patches}, nnz={pm.n_obs})")
