"""Per-CTA balance of the dictionary step's element phase (tuning build):
measured per-CTA element-phase time against the CTA's work (ELL positions, waves
by lanes-per-column, tiles), with a least-squares cost model.

  PB200_LIB_VARIANT=tune PB_DICT_PROF_CTAS=1 python tools/dict_balance.py [cfg] [epochs]
"""
import ctypes
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import bench  # noqa: E402
from paper_2311_15061_b200 import _lib  # noqa: E402
from paper_2311_15061_b200 import bpfa as gb  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402
from test_gpu_patches import _carve  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
E = int(sys.argv[2]) if len(sys.argv) > 2 else 5
TVC = float(os.environ.get("PB_DICT_TILE_COST", "500"))
cfg = bench.CFGS[cid]
img, mask = bench.config_inputs(cfg)
pm = pp.extract_patches(img, mask, pp.PatchSpec(cfg["patch"]), len(cfg["shape"]) == 2)
hp = gb.Hyperparams(num_atoms=cfg["k"])
st = gb.init_state(pm, hp, 0, "prior")
for _ in range(2):
    gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
lib = _lib.load()
lib.pb_dict_profile(1, None)
for _ in range(E):
    gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
out = (ctypes.c_double * 12)()
with tempfile.TemporaryFile(mode="w+") as f:
    sys.stderr.flush()
    saved = os.dup(2)
    os.dup2(f.fileno(), 2)
    try:
        lib.pb_dict_profile(0, out)
    finally:
        os.dup2(saved, 2)
        os.close(saved)
    f.seek(0)
    lines = [ln.split() for ln in f if ln.startswith("cta ")]
t_el = np.array([float(x[3]) for x in lines]) / E   # element phase, ms per sweep
t_fw = np.array([float(x[9]) for x in lines]) / E   # warp 0's tile-fill waits inside it
G = len(t_el)
if os.environ.get("PB_DICT_DEBUG", "0") == "32":   # reversed CTA <-> range map: index by range
    t_el = t_el[::-1].copy()
    t_fw = t_fw[::-1].copy()
print(f"fill waits (warp 0): mean {t_fw.mean():.4f} ms, cv {t_fw.std() / t_fw.mean():.3f}, "
      f"corr with element time {np.corrcoef(t_fw, t_el)[0, 1]:+.3f}; element time minus waits cv "
      f"{(t_el - t_fw).std() / (t_el - t_fw).mean():.3f}")
tag = os.environ.get("BALANCE_TAG")
if tag:
    os.makedirs("gpurun_out", exist_ok=True)
    np.save(f"gpurun_out/balance_cfg{cid}_{tag}.npy", t_el)

ix = pm.index()
b = _carve(pm._cache["ix_buf"].cpu().numpy(), pm.num_patches, pm.patch_size, int(ix.nnz))
eb = b["ell_base"].astype(np.int64)
wb = b["wave_base"].astype(np.int64)
woff = b["wave_off"].astype(np.int64)
meta = b["wave_meta"].astype(np.int64)
nt = len(eb) - 1
if tag and os.environ.get("BALANCE_DUMP"):   # the ELL index for offline analysis
    np.savez_compressed(f"gpurun_out/balance_cfg{cid}_index.npz", ell_base=eb, wave_base=wb,
                        wave_off=b["wave_off"][:wb[nt]], wave_meta=b["wave_meta"][:wb[nt]],
                        wave_col=b["wave_col"][:32 * wb[nt]], e_ell=b["e_ell"][:eb[nt]], t_el=t_el, tvc=TVC)
tot = eb[-1] + TVC * nt


def boundary(c):   # mirror of ell_cta_range (split_nearest off)
    if c <= 0:
        return 0
    if c >= G:
        return int(wb[nt])
    target = tot * c / G
    lo = int(np.searchsorted(eb[:nt] + TVC * np.arange(nt), target, side="right") - 1)
    over = target - (eb[lo] + TVC * lo) - TVC
    w0, w1 = wb[lo], wb[lo + 1]
    if over <= 0 or w1 == w0:
        return int(w0)
    ws = np.arange(w0, w1)
    return int(ws[np.searchsorted(woff[ws], over, side="right") - 1])


bd = [boundary(c) for c in range(G + 1)]
wave_tile = np.searchsorted(wb, np.arange(wb[nt]), side="right") - 1
feat = []
for c in range(G):
    w = np.arange(bd[c], bd[c + 1])
    lw = meta[w] & 0xFF
    lg = meta[w] >> 8
    row = [32.0 * lw.sum()]
    row += [float((lg == g).sum()) for g in range(6)]
    row += [float(len(np.unique(wave_tile[w]))) if len(w) else 0.0]
    feat.append(row)
X = np.array(feat)
names = ["positions"] + [f"waves lg{g}" for g in range(6)] + ["tiles"]
print(f"cfg{cid}: {G} CTAs, element phase per sweep: mean {t_el.mean():.4f} ms, min {t_el.min():.4f}, "
      f"max {t_el.max():.4f} (max/mean {t_el.max() / t_el.mean():.3f})")
print("slowest CTAs:", np.argsort(-t_el)[:8], "fastest:", np.argsort(t_el)[:4])
sys.stdout.flush()
for nm, col in zip(names, X.T):
    if col.std() > 0:
        print(f"  {nm:12s} mean {col.mean():12.1f}  cv {col.std() / col.mean():.3f}  "
              f"corr(t) {np.corrcoef(col, t_el)[0, 1]:+.3f}")
keep = [i for i in range(X.shape[1]) if X[:, i].std() > 0 or i == 0]
A = np.column_stack([X[:, keep], np.ones(G)])
coef, *_ = np.linalg.lstsq(A, t_el, rcond=None)
pred = A @ coef
print("fit (ms per unit):", {names[i]: f"{c:.3e}" for i, c in zip(keep, coef)}, f"const {coef[-1]:.4f}")
print(f"residual std {np.std(t_el - pred) * 1e3:.2f} us vs spread std {t_el.std() * 1e3:.2f} us")
pos_us = coef[0] * 1e3
for i, c in zip(keep, coef):
    print(f"  {names[i]:12s} = {c / coef[0]:10.1f} positions")
