"""Extraction / overlap-add timing on the 2-D BASELINE configs (CUDA events,
median of repeats) against their algorithmic HBM bytes:
  extract  read M*(8+1) (f64 frame + u8 mask), write N*P*(4+1) + N*8 (means, counts)
  OLA      read N*P*4 (estimates) + N*4 (means) + M*9 (DC: frame + mask), write M*8
python tools/patch_timing.py  [PB200_LIB_VARIANT=name]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6547.8
out = {}
for cid in (0, 1, 2, 4):
    cfg = bench.CFGS[cid]
    img, mask = bench.config_inputs(cfg)
    spec = pp.PatchSpec(cfg["patch"])
    t = torch.from_numpy(img).cuda()
    m = torch.from_numpy(mask.astype(np.uint8)).cuda()
    pm = pp.extract_patches(t, m, spec, True)
    est = pm.values_pn.clone()
    g = spec.desc(img.shape)
    import ctypes

    from paper_2311_15061_b200 import _lib

    lib = _lib.load()
    vals, obs = torch.empty_like(pm.values_pn), torch.empty_like(pm.observed_pn)
    means, counts = torch.empty_like(pm.means_dev), torch.empty_like(pm.counts)
    rec = torch.empty_like(t)
    st = torch.cuda.current_stream().cuda_stream
    res = {}
    # kernel launches through the C ABI on preallocated device buffers
    for name, fn in (("extract", lambda: lib.pb_extract_patches(ctypes.byref(g), t.data_ptr(), 1, m.data_ptr(), 1,
                                                                vals.data_ptr(), obs.data_ptr(), means.data_ptr(),
                                                                counts.data_ptr(), st)),
                     ("ola", lambda: lib.pb_reconstitute(ctypes.byref(g), est.data_ptr(), 1.0, pm.means_dev.data_ptr(),
                                                         t.data_ptr(), m.data_ptr(), 1, 1, rec.data_ptr(), None,
                                                         st))):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        M, N, P = img.size, pm.num_patches, pm.patch_size
        nbytes = M * 9 + N * P * 5 + N * 8 if name == "extract" else N * P * 4 + N * 4 + M * 9 + M * 8
        res[name] = {"ms": ms, "alg_bytes": nbytes, "gbs": nbytes / ms / 1e6, "frac": nbytes / ms / 1e6 / peak}
    out[f"configs[{cid}]"] = res
    print(cid, {k: (round(v["ms"], 4), round(v["frac"], 3)) for k, v in res.items()}, flush=True)
print(json.dumps(out))
