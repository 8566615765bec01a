"""Pin the oracle against golden fixtures produced by the reference itself.

The oracle (oracle/) is a restatement of reference patchbeam; these tests show
it reproduces the reference's outputs BIT-FOR-BIT (f64) on the committed
fixtures (tests/golden/make_golden.py ran the reference to make them).
"""

import numpy as np
import pytest

from oracle import bpfa as ob
from oracle import patches as op
from paper_2311_15061_b200 import inputs


def test_extract_reconstitute_bit_exact(golden):
    g = golden("extract_cases.npz")
    for ci in range(int(g["num_cases"])):
        p = f"c{ci}_"
        pm = op.extract_patches(g[p + "tensor"], g[p + "mask"], tuple(g[p + "patch"]),
                                tuple(g[p + "stride"]), bool(g[p + "mean_subtract"]))
        assert np.array_equal(pm.values, g[p + "values"]), ci
        assert np.array_equal(pm.observed, g[p + "observed"]), ci
        assert np.array_equal(pm.origins, g[p + "origins"]), ci
        assert np.array_equal(pm.means, g[p + "means"]), ci
        cov = op.coverage(pm.tensor_shape, pm.patch_shape, pm.stride)
        assert np.array_equal(cov, g[p + "coverage"]), ci
        rec = op.reconstitute(pm, g[p + "est"])
        assert np.array_equal(rec, g[p + "recon"]), ci


def test_strict_coverage_error(golden):
    g = golden("extract_cases.npz")
    p = "c7_"
    pm = op.extract_patches(g[p + "tensor"], g[p + "mask"], (2, 2), (2, 2), True)
    with pytest.raises(op.CoverageError):
        op.reconstitute(pm, pm.values, strict=True)


@pytest.mark.parametrize("name", ["small", "linehop", "frozen", "avg", "cfg1crop", "cube"])
def test_trajectory_bit_exact(golden, name):
    g = golden(f"traj_{name}.npz")
    patch = tuple(int(b) for b in g["patch"])
    pm = op.extract_patches(g["img"], g["mask"], patch, (), bool(g["mean_subtract"]))
    hp = ob.Hyper(num_atoms=int(g["k"]))
    seed = int(g["seed"])
    if "init_atoms" in g:
        st = ob.install_dictionary(seed, pm, hp, g["init_atoms"], g["init_pi"])
    else:
        st = ob.init_state(pm, hp, seed, init_mode=str(g["init_mode"]))
    assert np.array_equal(st.atoms, g["e0_atoms"])
    epochs = int(g["epochs"])
    avg = int(g["average_last"])
    tail = None
    for e in range(1, epochs + 1):
        ob.gibbs_epoch(st, pm, hp, freeze_dict=bool(g["freeze"]))
        assert np.array_equal(st.atoms, g[f"e{e}_atoms"]), (name, e, "atoms")
        assert np.array_equal(st.pi, g[f"e{e}_pi"]), (name, e, "pi")
        assert np.array_equal(st.usage, g[f"e{e}_usage"]), (name, e, "usage")
        assert np.array_equal(st.weights, g[f"e{e}_weights"]), (name, e, "weights")
        assert np.array_equal([st.gamma_s, st.gamma_eps], g[f"e{e}_gammas"]), (name, e)
        if e > epochs - avg:
            est = ob.compose_estimates(st)
            tail = est if tail is None else tail + est
    est = tail / avg
    assert np.array_equal(est, g["est"])
    rec = op.reconstitute(pm, est)
    assert np.array_equal(rec, g["recon"])
    assert np.array_equal(op.apply_data_consistency(rec, g["img"], g["mask"]), g["recon_dc"])


def test_posterior_helpers_bit_exact(golden):
    g = golden("posterior.npz")
    pm = op.extract_patches(g["img"], g["mask"], (3, 3), (), True)
    hp = ob.Hyper(num_atoms=5, concentration_a=1.3, concentration_b=0.7,
                  weight_shape=1.1, weight_rate=0.9, noise_shape=1.5, noise_rate=0.6)
    st = ob.State(atoms=g["atoms"].copy(), pi=g["pi"].copy(), usage=g["usage"].copy(),
                  weights=g["weights"].copy(), gamma_s=float(g["gammas"][0]),
                  gamma_eps=float(g["gammas"][1]), epoch=0, seed=4)
    for k in range(5):
        lam, mu = ob.atom_posterior(pm, st, k)
        assert np.array_equal(lam, g[f"k{k}_lam"]) and np.array_equal(mu, g[f"k{k}_mu"])
        lr, al, me = ob.code_posterior(pm, st, k)
        assert np.array_equal(lr, g[f"k{k}_logrho"])
        assert np.array_equal(al, g[f"k{k}_alpha"])
        assert np.array_equal(me, g[f"k{k}_mean"])
    a, b = ob.pi_posterior(st, hp)
    assert np.array_equal(a, g["pi_a"]) and np.array_equal(b, g["pi_b"])
    (ws, wr), (ns, nr) = ob.gamma_posteriors(pm, st, hp)
    assert np.array_equal([ws, wr, ns, nr], g["gamma_post"])


def test_input_generators_match_reference(golden):
    g = golden("masks.npz")
    specs = [((64, 64), 0.25, "uniform-random", 0), ((37, 53), 0.1, "uniform-random", 5),
             ((512, 512), 0.25, "line-hop", 0), ((30, 17), 0.33, "line-hop", 3),
             ((12, 10, 3), 0.2, "uniform-random", 1)]
    for i, (shape, ratio, kind, seed) in enumerate(specs):
        assert np.array_equal(inputs.make_mask(shape, ratio, kind, seed), g[f"m{i}"]), i
    assert np.array_equal(inputs.synthetic_texture((64, 64), seed=0), g["tex_64_s0"])
    assert np.array_equal(inputs.synthetic_texture((40, 56), seed=3, phase=0.45),
                          g["tex_40x56_s3_ph"])


def test_live_tail_oracle_matches_reference(golden):
    """Wire panels, residual maps and the adaptive sampler's exploit set
    (oracle/sampling.py) against the reference's own outputs."""
    from oracle import sampling as osm

    g = golden("live_tail.npz")
    for name in ("q2", "q3"):
        assert np.array_equal(osm.quantize_panel(g[f"{name}_in"]), g[f"{name}_out"]), name
    prev = None
    for t in range(3):
        assert np.array_equal(osm.residual_map(g[f"r{t}_recon"], prev), g[f"r{t}_resid"]), t
        prev = g[f"r{t}_recon"]
    for i in range(4):
        ratio, ef, _, _ = g[f"a{i}_spec"]
        res, mask = g[f"a{i}_res"], g[f"a{i}_mask"]
        budget, n_exploit = osm.adaptive_split(ratio, ef, res.size)
        assert int(mask.sum()) == budget
        ex = osm.adaptive_exploit(res, ratio, ef)
        assert len(ex) == n_exploit and mask.ravel()[ex].all(), i   # the exploit set is in the reference mask


def test_atlas_oracle_matches_reference(golden):
    from oracle import sampling as osm

    g = golden("atlas.npz")
    for name in ("a2", "a3", "a1", "a2sq"):
        c = osm.render_dictionary_atlas(g[f"{name}_atoms"], g[f"{name}_pi"], tuple(g[f"{name}_shape"]))
        assert np.array_equal(c, g[f"{name}_canvas"]), name


def test_live_pipeline_sequence_bit_exact(golden):
    """Pipeline.submit_frame (pipeline.py:217-276) over 3 warm-started frames,
    replayed by the oracle: codes re-burn each frame, dictionary / pi / gammas
    and the epoch counter carry over — reconstructions bit-exact."""
    g = golden("live.npz")
    hp = ob.Hyper(num_atoms=8)
    st = None
    for t in range(3):
        frame, mask = g[f"f{t}_frame"], g[f"f{t}_mask"]
        pm = op.extract_patches(frame, mask, (6, 6), (), True)
        if st is not None:
            st.usage[:] = False
            st.weights[:] = 0.0
        st, est = ob.infer(pm, hp, 2, 0, state=st)
        assert np.array_equal(op.reconstitute(pm, est), g[f"f{t}_recon"]), t
        assert np.array_equal(st.atoms, g[f"f{t}_atoms"]), t


def test_oracle_normalize_observed_matches_reference(golden):
    from oracle.cli import normalize_observed

    g = golden("entry.npz")
    for i in range(4):
        out, sc, off = normalize_observed(g[f"n{i}_frame"], g[f"n{i}_mask"])
        assert np.array_equal(out, g[f"n{i}_out"]), i
        assert (sc, off) == tuple(g[f"n{i}_scale_offset"]), i
