"""The INTEGRATION.md binding against the UNMODIFIED reference (baseline/_ref,
installed from /root/reference with pip; skipped when absent): the reference's
own Pipeline.submit_frame and its bpfa.infer inpaint flow run with their hot
path rebound to this library (paper_2311_15061_b200.integration.bind, replay
draws), and must reproduce the pure-reference results: per-frame
reconstruction within 1e-3, PSNR within 0.05 dB."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "patchbeam")),
                                 reason="reference not installed in baseline/_ref")]


@pytest.fixture(scope="module")
def patchbeam(tmp_path_factory):
    os.environ.setdefault("NUMBA_CACHE_DIR", str(tmp_path_factory.mktemp("numba")))
    sys.path.insert(0, REF)
    import patchbeam as pb
    import patchbeam.pipeline  # noqa: F401

    return pb


def _pipeline_run(pb, frames):
    from patchbeam import bpfa
    from patchbeam.patches import PatchSpec
    from patchbeam.pipeline import Pipeline, ProblemConfig
    from patchbeam.sampling import SamplerSpec

    pipe = Pipeline()
    cfg = ProblemConfig(name="p", patch_spec=PatchSpec((6, 6)), hyperparams=bpfa.Hyperparams(num_atoms=10),
                        sampler_spec=SamplerSpec(kind="line-hop", ratio=0.25, seed=0), epochs_per_frame=2, seed=0)
    h = pipe.create_problem(cfg)
    return [pipe.submit_frame(h, f, ground_truth=f) for f in frames]


def test_reference_pipeline_through_binding(cuda_device, patchbeam):
    from paper_2311_15061_b200 import inputs
    from paper_2311_15061_b200.integration import bind

    frames = inputs.synthetic_frames((40, 44), 3, seed=2)
    ref = _pipeline_run(patchbeam, frames)
    unbind = bind(patchbeam, rng="numpy")
    try:
        got = _pipeline_run(patchbeam, frames)
    finally:
        unbind()
    for r, g in zip(ref, got):
        assert np.array_equal(r.mask, g.mask)
        assert np.abs(g.reconstruction - r.reconstruction).max() <= 1e-3
        assert abs(g.metrics.psnr_db - r.metrics.psnr_db) <= 0.05
        assert g.metrics.epochs_run == r.metrics.epochs_run


def test_reference_inpaint_flow_through_binding(cuda_device, patchbeam):
    from patchbeam import bpfa, patches
    from patchbeam.sampling import SamplerSpec, make_mask

    from paper_2311_15061_b200 import inputs
    from paper_2311_15061_b200.integration import bind

    img = inputs.stem_lattice((64, 64), seed=3)
    mask = make_mask(SamplerSpec(kind="uniform-random", ratio=0.25, seed=3), img.shape)

    def flow():   # cmd_inpaint's steps (cli.py:247-274) through the reference modules
        pm = patches.extract_patches(img, mask, patches.PatchSpec((8, 8)), mean_subtract=True)
        _, est = bpfa.infer(pm, bpfa.Hyperparams(num_atoms=16), epochs=4, seed=7)
        return patches.apply_data_consistency(patches.reconstitute(pm, est), img, mask, True)

    ref = flow()
    unbind = bind(patchbeam, rng="numpy")
    try:
        got = flow()
    finally:
        unbind()
    assert np.abs(got - ref).max() <= 1e-3
