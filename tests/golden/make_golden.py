"""Generate golden fixtures by running the REFERENCE itself (build container only).

Usage (from the repo root, in the build container where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Imports ``patchbeam`` from /root/reference/pkg/src (read-only; the env vars keep
Numba's cache out of the reference tree) and writes small .npz files next to
this script.  The fixtures pin oracle/ (tests/test_oracle_golden.py) and the
CUDA path's index/bit-exact behaviour (tests/test_gpu_*.py).  Nothing on the
GPU box reads /root/reference; it only reads these committed fixtures.

Recorded environment goes into ``meta.json`` (numpy/numba/python versions).
"""

from __future__ import annotations

import json
import os
import platform
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import patchbeam  # noqa: F401
    return patchbeam


def extraction_cases(pb):
    from patchbeam.patches import PatchSpec, coverage_map, extract_patches, reconstitute

    rng = np.random.default_rng(20260101)
    cases = [
        ((4, 4), (2, 2), (2, 2), 1.0, False),
        ((9, 11), (3, 3), (1, 1), 0.5, True),
        ((10, 11), (3, 4), (2, 3), 0.3, True),
        ((17,), (4,), (3,), 0.6, False),
        ((6, 7, 5), (2, 3, 5), (1, 2, 1), 0.4, False),
        ((5, 4, 3, 4), (2, 2, 3, 2), (1, 2, 1, 1), 0.5, True),
        ((32, 32), (8, 8), (1, 1), 0.25, True),
        ((5, 5), (2, 2), (2, 2), 1.0, True),      # uncovered margin
        ((12, 12), (4, 4), (1, 1), 0.0, True),    # empty mask
    ]
    out = {}
    for ci, (shape, patch, stride, ratio, ms) in enumerate(cases):
        t = rng.random(shape)
        mask = rng.random(shape) < ratio
        pm = extract_patches(t, mask, PatchSpec(patch, stride), mean_subtract=ms)
        est = rng.standard_normal(pm.values.shape)
        rec = reconstitute(pm, est)
        pre = f"c{ci}_"
        out[pre + "tensor"] = t
        out[pre + "mask"] = mask
        out[pre + "patch"] = np.asarray(patch)
        out[pre + "stride"] = np.asarray(stride)
        out[pre + "mean_subtract"] = np.asarray(ms)
        out[pre + "values"] = pm.values
        out[pre + "observed"] = pm.observed
        out[pre + "origins"] = pm.origins
        out[pre + "means"] = pm.means
        out[pre + "coverage"] = coverage_map(pm)
        out[pre + "est"] = est
        out[pre + "recon"] = rec
    out["num_cases"] = np.asarray(len(cases))
    np.savez_compressed(os.path.join(OUT, "extract_cases.npz"), **out)


def _traj(pb, name, img_shape, patch, ratio, kind, k, epochs, seed, mask_seed,
          mean_subtract=True, freeze=False, init_mode="data", initial=False, average_last=1, cube_bands=0):
    from patchbeam import bpfa
    from patchbeam.patches import PatchSpec, extract_patches
    from patchbeam.sampling import SamplerSpec, make_mask
    from patchbeam.sources import synthetic_texture

    img = synthetic_texture(img_shape, seed=mask_seed)
    if cube_bands:  # hyperspectral-like cube (configs[3] shape class): texture x smooth spectrum
        spec = 0.5 + 0.5 * np.sin(np.linspace(0, 3 * np.pi, cube_bands))
        img = img[:, :, None] * spec[None, None, :]
    mask = make_mask(SamplerSpec(kind=kind, ratio=ratio, seed=mask_seed), img.shape)
    pm = extract_patches(img, mask, PatchSpec(patch), mean_subtract=mean_subtract)
    hp = bpfa.Hyperparams(num_atoms=k)
    if initial:
        r = np.random.default_rng(seed + 99)
        atoms = r.standard_normal((k, pm.patch_size))
        atoms /= np.linalg.norm(atoms, axis=1, keepdims=True)
        init = bpfa.Dictionary(atoms, r.uniform(0.2, 0.8, k), tuple(patch))
        state = bpfa.install_dictionary(seed, pm, hp, init)
        out_init = {"init_atoms": atoms, "init_pi": init.pi}
    else:
        state = bpfa.init_state(pm, hp, seed, init_mode=init_mode)
        out_init = {}
    rec = {"img": img, "mask": mask, "patch": np.asarray(patch), "k": np.asarray(k),
           "seed": np.asarray(seed), "epochs": np.asarray(epochs),
           "mean_subtract": np.asarray(mean_subtract), "freeze": np.asarray(freeze),
           "init_mode": np.asarray(init_mode), "average_last": np.asarray(average_last),
           "e0_atoms": state.dictionary.atoms.copy(), **out_init}
    tail = None
    for e in range(1, epochs + 1):
        bpfa.gibbs_epoch(state, pm, hp, freeze_dict=freeze)
        rec[f"e{e}_atoms"] = state.dictionary.atoms.copy()
        rec[f"e{e}_pi"] = state.dictionary.pi.copy()
        rec[f"e{e}_usage"] = state.usage.copy()
        rec[f"e{e}_weights"] = state.weights.copy()
        rec[f"e{e}_gammas"] = np.array([state.weight_precision, state.noise_precision])
        if e > epochs - average_last:
            est = bpfa.compose_estimates(state)
            tail = est if tail is None else tail + est
    rec["est"] = tail / average_last
    from patchbeam.patches import apply_data_consistency, reconstitute
    rec["recon"] = reconstitute(pm, rec["est"])
    rec["recon_dc"] = apply_data_consistency(rec["recon"], img, mask, True)
    np.savez_compressed(os.path.join(OUT, f"traj_{name}.npz"), **rec)


def trajectories(pb):
    _traj(pb, "small", (24, 24), (4, 4), 0.4, "uniform-random", 6, 4, 3, 5)
    _traj(pb, "linehop", (32, 40), (8, 8), 0.25, "line-hop", 8, 3, 7, 2)
    _traj(pb, "frozen", (20, 20), (5, 5), 0.3, "uniform-random", 4, 3, 11, 4,
          freeze=True, initial=True)
    _traj(pb, "avg", (16, 20), (3, 3), 0.5, "uniform-random", 5, 4, 13, 6,
          mean_subtract=False, average_last=2, init_mode="prior")
    _traj(pb, "cfg1crop", (48, 48), (8, 8), 0.25, "uniform-random", 16, 3, 0, 0)
    _traj(pb, "cube", (14, 16), (4, 4, 3), 0.2, "uniform-random", 8, 3, 21, 8, mean_subtract=False,
          cube_bands=6)


def masks(pb):
    from patchbeam.sampling import SamplerSpec, make_mask
    from patchbeam.sources import synthetic_texture

    out = {}
    specs = [((64, 64), 0.25, "uniform-random", 0), ((37, 53), 0.1, "uniform-random", 5),
             ((512, 512), 0.25, "line-hop", 0), ((30, 17), 0.33, "line-hop", 3),
             ((12, 10, 3), 0.2, "uniform-random", 1)]
    for i, (shape, ratio, kind, seed) in enumerate(specs):
        out[f"m{i}"] = make_mask(SamplerSpec(kind=kind, ratio=ratio, seed=seed), shape)
        out[f"m{i}_spec"] = np.array([str(shape), str(ratio), kind, str(seed)])
    out["tex_64_s0"] = synthetic_texture((64, 64), seed=0)
    out["tex_40x56_s3_ph"] = synthetic_texture((40, 56), seed=3, phase=0.45)
    np.savez_compressed(os.path.join(OUT, "masks.npz"), **out)


def live(pb):
    """Pipeline.submit_frame over 3 synthetic frames (warm start, K=8)."""
    from patchbeam import bpfa
    from patchbeam.pipeline import Pipeline, ProblemConfig
    from patchbeam.patches import PatchSpec
    from patchbeam.sampling import SamplerSpec
    from patchbeam.sources import SyntheticSource

    pipe = Pipeline()
    cfg = ProblemConfig(name="p", patch_spec=PatchSpec((6, 6)),
                        hyperparams=bpfa.Hyperparams(num_atoms=8),
                        sampler_spec=SamplerSpec(kind="line-hop", ratio=0.25, seed=0),
                        epochs_per_frame=2, seed=0)
    h = pipe.create_problem(cfg)
    src = SyntheticSource((32, 32), num_frames=3, seed=0)
    out = {}
    for t, frame in enumerate(src.frames()):
        res = pipe.submit_frame(h, frame, ground_truth=frame)
        out[f"f{t}_frame"] = frame
        out[f"f{t}_recon"] = res.reconstruction
        out[f"f{t}_mask"] = res.mask
        out[f"f{t}_atoms"] = res.dictionary.atoms
        out[f"f{t}_psnr"] = np.asarray(res.metrics.psnr_db)
    np.savez_compressed(os.path.join(OUT, "live.npz"), **out)


def posterior(pb):
    """Conditional parameters on random states (reference helpers bpfa.py:189-235)."""
    from patchbeam import bpfa
    from patchbeam.patches import PatchSpec, extract_patches

    rng = np.random.default_rng(77)
    img = rng.random((10, 9))
    mask = rng.random(img.shape) < 0.6
    pm = extract_patches(img, mask, PatchSpec((3, 3)), mean_subtract=True)
    hp = bpfa.Hyperparams(num_atoms=5, concentration_a=1.3, concentration_b=0.7,
                          weight_shape=1.1, weight_rate=0.9, noise_shape=1.5, noise_rate=0.6)
    st = bpfa.init_state(pm, hp, seed=4, init_mode="prior")
    n, k = st.usage.shape
    st.usage[:] = rng.random((n, k)) < 0.5
    st.weights[:] = rng.standard_normal((n, k))
    st.dictionary.atoms[:] = rng.standard_normal(st.dictionary.atoms.shape)
    st.dictionary.pi = rng.uniform(0.05, 0.95, size=k)
    st.weight_precision = 1.7
    st.noise_precision = 23.0
    out = {"img": img, "mask": mask, "usage": st.usage, "weights": st.weights,
           "atoms": st.dictionary.atoms, "pi": st.dictionary.pi,
           "gammas": np.array([st.weight_precision, st.noise_precision])}
    for kk in range(k):
        lam, mu = bpfa.atom_posterior(pm, st, kk)
        lr, al, me = bpfa.code_posterior(pm, st, kk)
        out[f"k{kk}_lam"], out[f"k{kk}_mu"] = lam, mu
        out[f"k{kk}_logrho"], out[f"k{kk}_alpha"], out[f"k{kk}_mean"] = lr, al, me
    a, b = bpfa.pi_posterior(st, hp)
    (ws, wr), (ns, nr) = bpfa.gamma_posteriors(pm, st, hp)
    out["pi_a"], out["pi_b"] = a, b
    out["gamma_post"] = np.array([ws, wr, ns, nr])
    np.savez_compressed(os.path.join(OUT, "posterior.npz"), **out)


def live_tail(pb):
    """The live path's tail: uint8 wire panels (server.py:46-53), the residual
    map of consecutive reconstructions (pipeline.py:265-269) and the
    adaptive-residual sampler (sampling.py:184-207)."""
    from patchbeam import bpfa
    from patchbeam.patches import PatchSpec
    from patchbeam.pipeline import Pipeline, ProblemConfig
    from patchbeam.sampling import SamplerSpec, run_strategy
    from patchbeam.server import quantize_panel
    from patchbeam.sources import SyntheticSource

    rng = np.random.default_rng(515)
    out = {}
    # panels: out-of-range values, exact half-steps (round half to even), rank 3
    p2 = rng.uniform(-0.2, 1.2, size=(9, 13))
    p2[0, :6] = (np.arange(6) + 0.5) / 255.0
    p3 = rng.uniform(0, 1, size=(7, 5, 3))
    for name, pnl in (("q2", p2), ("q3", p3)):
        out[f"{name}_in"] = pnl
        out[f"{name}_out"] = quantize_panel(pnl)
    # adaptive sampler on maps with ties (integer-valued residuals)
    cases = [((24, 20), 0.25, 0.5, 0), ((16, 16), 0.1, 0.75, 3), ((12, 10, 3), 0.3, 0.4, 1), ((30, 30), 0.2, 1.0, 2)]
    for i, (shape, ratio, ef, seed) in enumerate(cases):
        res = rng.integers(0, 6, size=shape).astype(np.float64) * 0.25
        spec = SamplerSpec(kind="adaptive-residual", ratio=ratio, seed=seed, parameters={"exploit_fraction": ef})
        out[f"a{i}_res"] = res
        out[f"a{i}_mask"] = run_strategy(spec, shape, prev_mask=None, residual_map=res, frame_index=i)
        out[f"a{i}_spec"] = np.array([ratio, ef, seed, i], dtype=np.float64)
    # residual maps of a 3-frame live run (DC off: the recon is pre-consistency)
    pipe = Pipeline()
    cfg = ProblemConfig(name="r", patch_spec=PatchSpec((6, 6)), hyperparams=bpfa.Hyperparams(num_atoms=8),
                        sampler_spec=SamplerSpec(kind="uniform-random", ratio=0.3, seed=0),
                        epochs_per_frame=2, seed=0, data_consistency=False)
    h = pipe.create_problem(cfg)
    for t, frame in enumerate(SyntheticSource((24, 24), num_frames=3, seed=0).frames()):
        res = pipe.submit_frame(h, frame)
        out[f"r{t}_recon"] = res.reconstruction
        out[f"r{t}_resid"] = h.residual_map.copy()
    np.savez_compressed(os.path.join(OUT, "live_tail.npz"), **out)


def dict_files(pb):
    """SADF dictionary files written by the reference (formats.py:147-161)."""
    from patchbeam.bpfa import Dictionary
    from patchbeam.formats import write_dict

    rng = np.random.default_rng(99)
    d = Dictionary(atoms=rng.standard_normal((6, 12)), pi=rng.uniform(0, 1, 6), patch_shape=(3, 4))
    write_dict(os.path.join(OUT, "dict_k6_3x4.sadf"), d)
    write_dict(os.path.join(OUT, "dict_k6_3x4_nopi.sadf"), d, include_pi=False)
    np.savez_compressed(os.path.join(OUT, "dict_src.npz"), atoms=d.atoms, pi=d.pi)


def atlases(pb):
    """server.render_dictionary_atlas (server.py:84-120) on f32-exact atoms:
    pi ties, a constant atom, ranks 1-3."""
    from patchbeam.bpfa import Dictionary
    from patchbeam.server import render_dictionary_atlas

    rng = np.random.default_rng(404)
    out = {}
    for name, k, shape in (("a2", 10, (4, 5)), ("a3", 7, (3, 4, 2)), ("a1", 5, (6,)), ("a2sq", 16, (3, 3))):
        p = int(np.prod(shape))
        atoms = rng.standard_normal((k, p)).astype(np.float32).astype(np.float64)
        atoms[1] = 0.25                                    # constant atom -> mid-grey
        pi = np.round(rng.uniform(0, 1, k), 1)             # ties broken by atom index
        d = Dictionary(atoms=atoms, pi=pi, patch_shape=shape)
        out[f"{name}_atoms"], out[f"{name}_pi"] = atoms, pi
        out[f"{name}_shape"] = np.asarray(shape)
        out[f"{name}_canvas"] = render_dictionary_atlas(d)
    np.savez_compressed(os.path.join(OUT, "atlas.npz"), **out)


def entry_cases(pb):
    """The CLI entry flows' steps (cli.py): _normalize_observed cases, an inpaint
    of an out-of-range frame (cmd_inpaint's steps), a learn over two images
    (cmd_learn's steps), and a transfer_dictionary onto an extended patch shape."""
    from patchbeam import bpfa
    from patchbeam.cli import _normalize_observed
    from patchbeam.patches import PatchMatrix, PatchSpec, apply_data_consistency, extract_patches, reconstitute
    from patchbeam.sampling import SamplerSpec, make_mask

    rng = np.random.default_rng(606)
    out = {}
    frames = [rng.random((9, 11)),                                   # already in [0, 1]: identity
              rng.random((9, 11)) * 7.0 - 2.0,                       # affine
              np.full((9, 11), 3.5),                                 # constant observed values
              rng.random((9, 11)) * 4.0 + 1.0]                       # mask empty -> identity
    masks = [rng.random((9, 11)) < 0.4, rng.random((9, 11)) < 0.4, rng.random((9, 11)) < 0.4,
             np.zeros((9, 11), bool)]
    frames[1][~masks[1]] = 1e6                                       # unobserved garbage must not matter
    for i, (f, m) in enumerate(zip(frames, masks)):
        g, sc, off = _normalize_observed(f, m)
        out[f"n{i}_frame"], out[f"n{i}_mask"], out[f"n{i}_out"] = f, m, g
        out[f"n{i}_scale_offset"] = np.array([sc, off])
    # inpaint (cli.py:247-274): normalize -> extract (mean-sub) -> infer -> OLA -> DC
    img = rng.random((30, 28)) * 5.0 + 10.0
    mask = make_mask(SamplerSpec(kind="uniform-random", ratio=0.3, seed=3), img.shape)
    f, sc, off = _normalize_observed(img, mask)
    pm = extract_patches(f, mask, PatchSpec((5, 5)), mean_subtract=True)
    st, est = bpfa.infer(pm, bpfa.Hyperparams(num_atoms=12), epochs=3, seed=4)
    rec = apply_data_consistency(reconstitute(pm, est), f, mask, True)
    out.update(inp_img=img, inp_mask=mask, inp_recon=rec, inp_scale_offset=np.array([sc, off]),
               inp_atoms=st.dictionary.atoms)
    # learn (cli.py:342-386): masks keyed by seed + i, concatenated patch matrices, infer
    imgs = [rng.random((20, 22)), rng.random((18, 25))]
    seed, ratio = 5, 0.35
    parts = []
    for i, im in enumerate(imgs):
        mk = make_mask(SamplerSpec(ratio=ratio, seed=seed + i), im.shape)
        parts.append(extract_patches(im, mk, PatchSpec((4, 4)), mean_subtract=True))
    cat = PatchMatrix(values=np.concatenate([q.values for q in parts]),
                      observed=np.concatenate([q.observed for q in parts]),
                      origins=np.concatenate([q.origins for q in parts]),
                      means=np.concatenate([q.means for q in parts]),
                      tensor_shape=parts[0].tensor_shape, spec=PatchSpec((4, 4)), mean_subtracted=True)
    st, _ = bpfa.infer(cat, bpfa.Hyperparams(num_atoms=7), epochs=3, seed=seed)
    out.update(learn_img0=imgs[0], learn_img1=imgs[1], learn_atoms=st.dictionary.atoms, learn_pi=st.dictionary.pi,
               learn_n=np.asarray(cat.num_patches))
    # transfer_dictionary onto an extended patch shape (bpfa.py:417-458)
    src = bpfa.Dictionary(rng.standard_normal((5, 12)).astype(np.float32).astype(np.float64),
                          rng.uniform(0, 1, 5), (3, 4))
    src.atoms[2] = 0.0
    moved = bpfa.transfer_dictionary(src, (3, 4, 3), (10, 12, 3))
    out.update(tr_src=src.atoms, tr_pi=src.pi, tr_out=moved.atoms)
    np.savez_compressed(os.path.join(OUT, "entry.npz"), **out)


def main():
    pb = _import_reference()
    import numba

    only = sys.argv[1:]
    for name, fn in (("extract", extraction_cases), ("traj", trajectories), ("masks", masks), ("live", live),
                     ("posterior", posterior), ("live_tail", live_tail), ("dicts", dict_files),
                     ("atlas", atlases), ("entry", entry_cases)):
        if not only or name in only:
            fn(pb)
    meta = {"python": platform.python_version(), "numpy": np.__version__,
            "numba": numba.__version__, "reference": REF,
            "note": "generated by running the reference patchbeam package itself"}
    with open(os.path.join(OUT, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
