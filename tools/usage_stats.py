"""Sparsity of the code matrix Z over the sweep (bench configs[1] and configs[2]):
density, active atoms per patch, share of all-zero 8-atom blocks per patch."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_15061_b200 import bpfa as gb  # noqa: E402
from paper_2311_15061_b200 import inputs  # noqa: E402
from paper_2311_15061_b200 import patches as pp  # noqa: E402


def stats(st, n):
    z = st.usage_kn[:, :n].to(torch.float32)          # (K, N)
    k = z.shape[0]
    act = z.sum(0)
    blk = z[: k // 8 * 8].reshape(k // 8, 8, n).amax(1)   # (K/8, N)
    m = z.sum(1)
    return (f"density={z.mean().item():.4f} active/patch mean={act.mean().item():.1f} "
            f"p50={act.median().item():.0f} max={act.max().item():.0f} zero8blk={1 - blk.mean().item():.3f} "
            f"atoms_used={(m > 0).sum().item()} atoms>1%={(m > 0.01 * n).sum().item()}")


for name, cfg in (("configs[1]", bench.CFG), ("configs[2]", bench.LIVE)):
    if name == "configs[1]":
        img, mask = bench.workload_inputs(cfg)
    else:
        img = inputs.synthetic_frames(cfg["shape"], 1, seed=0)[0]
        mask = inputs.make_mask(cfg["shape"], cfg["ratio"], cfg["kind"], cfg["seed"])
    pm = pp.extract_patches(img, mask, pp.PatchSpec(cfg["patch"]), True)
    hp = gb.Hyperparams(num_atoms=cfg["k"])
    st = gb.init_state(pm, hp, cfg["seed"], "prior")
    for e in range(1, 51):
        gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
        if e in (1, 2, 3, 5, 8, 13, 20, 30, 50):
            print(name, "epoch", e, stats(st, pm.num_patches), flush=True)
