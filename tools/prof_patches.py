"""Profiling driver (under ncu): one extraction and one overlap-add of configs[1] (2-D tiled kernels)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = bench.CFGS[cid]
img, mask = bench.config_inputs(cfg)
t = torch.from_numpy(img).cuda()
m = torch.from_numpy(mask.astype(np.uint8)).cuda()
pm = pp.extract_patches(t, m, pp.PatchSpec(cfg["patch"]), True)
rec = pp.reconstitute(pm, pm.values_pn.T, dc_original=t, dc_mask=m, out="device")
torch.cuda.synchronize()
print("ok", pm.num_patches)
