import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import bench
from paper_2311_15061_b200 import patches as pp
from test_gpu_patches import _carve
cfg = bench.CFGS[1]
img, mask = bench.config_inputs(cfg)
pm = pp.extract_patches(img, mask, pp.PatchSpec(cfg["patch"]), True)
ix = pm.index()
b = _carve(pm._cache["ix_buf"].cpu().numpy(), pm.num_patches, pm.patch_size, int(ix.nnz))
eb = b["ell_base"].astype(np.int64); wb = b["wave_base"].astype(np.int64); woff = b["wave_off"].astype(np.int64)
meta = b["wave_meta"].astype(np.int64)
nt = len(eb) - 1; G = 148; tvc = 3000.0
tot = eb[-1] + tvc * nt
cost = lambda t: eb[t] + tvc * t
def boundary(c):
    if c <= 0: return 0
    if c >= G: return wb[nt]
    target = tot * c / G
    lo = np.searchsorted(eb + tvc * np.arange(nt + 1), target, side="right") - 1
    lo = min(lo, nt - 1)
    over = target - cost(lo) - tvc
    w0, w1 = wb[lo], wb[lo + 1]
    if over <= 0 or w1 == w0: return w0
    ws = np.arange(w0, w1)
    return ws[np.searchsorted(woff[ws], over, side="right") - 1]
bd = [boundary(c) for c in range(G + 1)]
pos = []
for c in range(G):
    lw = meta[bd[c]:bd[c + 1]] & 0xFF
    pos.append(int((32 * lw).sum()))
pos = np.array(pos)
print("nnz", ix.nnz, "ell", eb[-1], "pad %.3f" % (eb[-1] / ix.nnz - 1))
print("positions per CTA: mean %.0f min %d max %d; last 4:" % (pos.mean(), pos.min(), pos.max()), pos[-4:], "first 4:", pos[:4])
print("waves per CTA last:", bd[-1] - bd[-2], "mean", np.mean(np.diff(bd)))
R = 1 << (meta >> 8)
print("R histogram:", np.unique(R, return_counts=True))
print("Lw mean", (meta & 0xFF).mean(), "last CTA Lw mean", (meta[bd[-2]:bd[-1]] & 0xFF).mean())
