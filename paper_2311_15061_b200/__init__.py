"""paper_2311_15061_b200 — B200-native BPFA Gibbs-sampling inpainting hot path.

Drop-in for the train/inpaint path of the reference ``patchbeam`` package
(arXiv 2311.15061 "SenseAI"): the same public names as patchbeam/__init__.py:9-32
for the hot path, backed by hand-written sm_100a CUDA kernels behind a C ABI
(include/pb200.h, built in-tree to paper_2311_15061_b200/_lib/libpb200.so).
"""

from .bpfa import (  # noqa: F401
    Dictionary,
    DivergenceError,
    GibbsState,
    Hyperparams,
    compose_estimates,
    gibbs_epoch,
    infer,
    init_state,
    install_dictionary,
    transfer_dictionary,
)
from .entry import inpaint, learn, normalize_observed  # noqa: F401
from .live import LiveFrame, LiveProblem, adaptive_mask, transfer_between  # noqa: F401
from .patches import (  # noqa: F401
    CoverageError,
    PatchMatrix,
    PatchSpec,
    ShapeError,
    apply_data_consistency,
    coverage_map,
    extract_patches,
    normalize,
    reconstitute,
)

__version__ = "0.1.0"
