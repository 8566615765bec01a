"""Adaptive-mask timing (pb_adaptive_mask through the C ABI on a device residual
map; CUDA events, median of 20) at the live frame (512²) and configs[1] (1024²)
sizes.  PB200_LIB_VARIANT=name times another build of the library."""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_15061_b200 import _lib  # noqa: E402

lib = _lib.load()
out = {}
for shape in ((512, 512), (1024, 1024), (4096, 4096)):
    r = torch.rand(shape, dtype=torch.float64, device="cuda") * (torch.rand(shape, device="cuda") < 0.5)
    mask = torch.empty(shape, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    status = ctypes.c_int32(0)

    def call():
        rc = lib.pb_adaptive_mask(ctypes.c_void_p(r.data_ptr()), ctypes.c_int64(r.numel()), ctypes.c_double(0.1),
                                  ctypes.c_double(0.5), ctypes.c_uint64(3), ctypes.c_int64(7),
                                  ctypes.c_void_p(mask.data_ptr()), ctypes.byref(status), ctypes.c_void_p(st))
        assert rc == 0, _lib.last_error() if hasattr(_lib, "last_error") else rc

    for _ in range(3):
        call()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[f"{shape[0]}x{shape[1]}"] = {"ms": float(np.median(ts)), "selected": int(mask.sum())}
print(json.dumps(out))
