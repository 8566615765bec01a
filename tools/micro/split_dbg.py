import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2311_15061_b200 import inputs, patches as pp
for shape in [(128, 128), (300, 300)]:
    img = inputs.synthetic_texture(shape, seed=0)
    mask = inputs.make_mask(shape, 0.10, "uniform-random", 0)
    pm = pp.extract_patches(img, mask, pp.PatchSpec((10, 10)), True)
    ix = pm.index()
    torch.cuda.synchronize()
    print(shape, "cmax", ix.cmax, "split", ix.split_count, "nout", ix.n_outliers, flush=True)
