"""Run N live frames (BASELINE configs[2]) through pb_problem_submit_frame, for
launch lists / profiles of the live path:  python tools/live_frames.py [N]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_15061_b200 import _lib, inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
L = bench.LIVE
lib = _lib.load()
frames = inputs.synthetic_frames(L["shape"], n, seed=0)
mask = inputs.make_mask(L["shape"], L["ratio"], L["kind"], L["seed"]).astype(np.uint8)
fh = [torch.from_numpy(f).pin_memory() for f in frames]
lm = torch.from_numpy(mask).pin_memory()
lo = torch.empty(L["shape"], dtype=torch.float64).pin_memory()
pr = ctypes.c_void_p()
_lib.check(lib.pb_problem_create(ctypes.byref(bench.problem_desc(L, L["epochs"], warm=True, dc=False)), ctypes.byref(pr)))
for f in fh:
    _lib.check(lib.pb_problem_submit_frame(pr, f.data_ptr(), lm.data_ptr(), lo.data_ptr()))
    print(f"frame gpu ms {lib.pb_problem_last_gpu_ms(pr):.3f}")
lib.pb_problem_destroy(pr)
