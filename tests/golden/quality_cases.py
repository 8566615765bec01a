"""Reconstruction-quality cases shared by tests/golden/make_quality.py (the
reference side, build container), tests/test_gpu_quality.py and bench.py's
``quality`` key (the device side, GPU box).  Inputs only: nothing here imports
the reference or the oracle.

``run_device`` runs a case through this package's public API exactly as the
reference CLI / Pipeline would (cli.py:247-274 ``inpaint``; pipeline.py:217-251
``submit_frame`` warm start) and returns per-frame (psnr, ssim).
"""

from __future__ import annotations

import numpy as np

SEEDS = (0, 1, 2)

CASES = {
    "cfg0": dict(what="configs[0] full: 256x256 STEM-like, 25% uniform, 8x8, K=64, 10 epochs, CLI inpaint "
                      "(mean subtraction, data consistency on)",
                 shape=(256, 256), ratio=0.25, kind="uniform-random", patch=(8, 8), k=64, epochs=10),
    "cfg1crop": dict(what="configs[1] crop: top-left 192x192 of the 1024x1024 STEM-like frame and its 10% "
                          "uniform mask, 10x10, K=256, 50 epochs, CLI inpaint (DC on)",
                     shape=(1024, 1024), crop=192, ratio=0.10, kind="uniform-random", patch=(10, 10), k=256,
                     epochs=50),
    "cfg2": dict(what="configs[2] live: 3 synthetic 512x512 frames, 25% line-hop, 8x8, K=256, 2 warm-started "
                      "epochs/frame, Pipeline defaults (DC off)",
                 shape=(512, 512), ratio=0.25, kind="line-hop", patch=(8, 8), k=256, epochs=2, frames=3),
}


def case_inputs(name):
    """Frame(s) and mask of a quality case."""
    from paper_2311_15061_b200 import inputs

    c = CASES[name]
    mask = inputs.make_mask(c["shape"], c["ratio"], c["kind"], 0)
    if name == "cfg2":
        return inputs.synthetic_frames(c["shape"], c["frames"], seed=0), mask
    img = inputs.stem_lattice(c["shape"], seed=0)
    if "crop" in c:
        s = c["crop"]
        img, mask = np.ascontiguousarray(img[:s, :s]), np.ascontiguousarray(mask[:s, :s])
    return img, mask


def run_device(name, seed, rng="philox", return_recon=False):
    """The case on the device through the public API -> list of (psnr, ssim) per frame."""
    from paper_2311_15061_b200 import bpfa as gb
    from paper_2311_15061_b200 import patches as pp
    from paper_2311_15061_b200.live import LiveProblem
    from paper_2311_15061_b200.metrics import psnr, ssim

    c = CASES[name]
    if name == "cfg2":
        frames, mask = case_inputs(name)
        out, recs = [], []
        with LiveProblem(c["shape"], pp.PatchSpec(c["patch"]), gb.Hyperparams(num_atoms=c["k"]), seed=seed,
                         epochs_per_frame=c["epochs"], rng=rng) as lp:
            for f in frames:
                r = lp.submit_frame(f, mask).reconstruction
                out.append((psnr(r, f), ssim(r, f)))
                recs.append(r)
        return (out, recs) if return_recon else out
    img, mask = case_inputs(name)
    pm = pp.extract_patches(img, mask, pp.PatchSpec(c["patch"]), True)
    _, est = gb.infer(pm, gb.Hyperparams(num_atoms=c["k"]), c["epochs"], seed, rng=rng)
    rec = pp.reconstitute(pm, est, dc_original=img, dc_mask=mask)
    out = [(psnr(rec, img), ssim(rec, img))]
    return (out, [rec]) if return_recon else out


def reference_summary(qjson, name):
    """Mean / std over seeds (and frames) of the reference's recorded PSNR / SSIM."""
    runs = qjson[name]["runs"]
    p = np.array([np.atleast_1d(r["psnr_db"]) for r in runs], dtype=np.float64)
    s = np.array([np.atleast_1d(r["ssim"]) for r in runs], dtype=np.float64)
    return p, s
