"""Route the reference package's hot path to this library in place — the
binding INTEGRATION.md describes, as code (and exercised by
tests/test_gpu_integration.py against the UNMODIFIED reference installed in
baseline/_ref).

``bind(patchbeam)`` rebinds, in the reference's own modules, the names its
train / inpaint / live callers look up (``bpfa.infer`` through the module object,
pipeline.py:23 and cli.py:247-274; the ``patches`` functions pipeline.py imported
by name, pipeline.py:27-33; ``model_stats`` for device state, metrics.py:43-51) to
this package's device implementations; reference ``PatchSpec`` / ``Hyperparams``
/ ``Dictionary`` objects are accepted as they are.  Returns an ``unbind()``.
"""

from __future__ import annotations

from . import bpfa as _b
from . import patches as _p


def bind(patchbeam, rng: str = "numpy"):
    import importlib

    pb_bpfa = importlib.import_module(patchbeam.__name__ + ".bpfa")
    pb_patches = importlib.import_module(patchbeam.__name__ + ".patches")
    pb_pipeline = importlib.import_module(patchbeam.__name__ + ".pipeline")
    pb_metrics = importlib.import_module(patchbeam.__name__ + ".metrics")

    def spec_of(spec):
        return _p.PatchSpec(tuple(spec.patch_shape), tuple(spec.stride))

    def extract_patches(tensor, mask, spec, mean_subtract=False):
        return _p.extract_patches(tensor, mask, spec_of(spec), mean_subtract)

    def reconstitute(pm, estimates, strict=False):
        return _p.reconstitute(pm, estimates, strict)

    def infer(pm, hp, epochs, seed, freeze_dict=False, initial_dict=None, init_mode="data", average_last=1,
              state=None):
        return _b.infer(pm, hp, epochs, seed, freeze_dict=freeze_dict, initial_dict=initial_dict,
                        init_mode=init_mode, average_last=average_last, state=state, rng=rng)

    def gibbs_epoch(state, pm, hp, freeze_dict=False):
        return _b.gibbs_epoch(state, pm, hp, freeze_dict=freeze_dict, rng=rng)

    def model_stats(state):
        h = state.dictionary.to_host()
        return (float(state.usage.sum()) / state.num_patches, h.pi.copy(), state.weight_precision,
                state.noise_precision)

    table = [
        (pb_patches, "extract_patches", extract_patches), (pb_patches, "reconstitute", reconstitute),
        (pb_pipeline, "extract_patches", extract_patches), (pb_pipeline, "reconstitute", reconstitute),
        (pb_bpfa, "infer", infer), (pb_bpfa, "gibbs_epoch", gibbs_epoch),
        (pb_bpfa, "init_state", _b.init_state), (pb_bpfa, "compose_estimates", _b.compose_estimates),
        (pb_bpfa, "install_dictionary", _b.install_dictionary),
        (pb_metrics, "model_stats", model_stats), (pb_pipeline, "model_stats", model_stats),
    ]
    saved = [(mod, name, getattr(mod, name)) for mod, name, _ in table]
    for mod, name, fn in table:
        setattr(mod, name, fn)

    def unbind():
        for mod, name, fn in saved:
            setattr(mod, name, fn)

    return unbind
