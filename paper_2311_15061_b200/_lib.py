"""ctypes binding of the sm_100a C-ABI library (include/pb200.h -> _lib/libpb200.so).

There is deliberately no CPU fallback: if the library is missing this module
raises, and every compute entry point needs a CUDA device (PB_ECUDA otherwise).
ctypes releases the GIL for the duration of each call.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PB200_LIB_VARIANT=name loads _lib/variants/libpb200_<name>.so (kernel-tuning experiments)
_VARIANT = os.environ.get("PB200_LIB_VARIANT")
LIB_PATH = os.path.join(_HERE, "_lib", "variants", f"libpb200_{_VARIANT}.so") if _VARIANT else \
    os.path.join(_HERE, "_lib", "libpb200.so")

PB_OK = 0
PB_ESHAPE = -1
PB_EVALUE = -2
PB_ECOVERAGE = -3
PB_EDIVERGED = -4
PB_ECUDA = -5
PB_EUNSUPPORTED = -6

PB_RESID_RECOMPUTE = 0
PB_RESID_FROM_VALUES = 1
PB_RESID_CARRY = 2

PB_RNG_REPLAY = 0
PB_RNG_PHILOX = 1

c_i32, c_i64, c_u64, c_f32, c_f64, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                          ctypes.c_float, ctypes.c_double, ctypes.c_void_p)


class GridDesc(ctypes.Structure):
    _fields_ = [("rank", c_i32), ("tensor_shape", c_i64 * 4), ("patch_shape", c_i32 * 4),
                ("stride", c_i32 * 4)]


class Scalars(ctypes.Structure):
    _fields_ = [("gamma_s", c_f64), ("gamma_eps", c_f64), ("sq_w", c_f64), ("sq_r", c_f64),
                ("epoch", c_i32), ("diverged", c_i32)]


class PatchIndex(ctypes.Structure):
    _fields_ = [("n", c_i64), ("p", c_i32), ("ntiles", c_i32), ("nnz", c_i64), ("cmax", c_i32),
                ("buffer", c_vp), ("split_count", c_i32), ("split_request", c_i32), ("n_outliers", c_i64),
                ("nnz_ell", c_i64)]


ALLREDUCE_FN = ctypes.CFUNCTYPE(c_i32, c_vp, c_vp, c_i64, c_i32, c_vp)


class EpochDesc(ctypes.Structure):
    _fields_ = [("n", c_i64), ("ld", c_i64), ("p", c_i32), ("k", c_i32), ("freeze_dict", c_i32), ("rng_mode", c_i32),
                ("resid_mode", c_i32), ("seed", c_u64), ("n_obs", c_i64), ("hyper", c_f64 * 6),
                ("values", c_vp), ("observed", c_vp), ("counts", c_vp), ("index", ctypes.POINTER(PatchIndex)),
                ("atoms", c_vp), ("pi", c_vp), ("usage", c_vp),
                ("weights", c_vp), ("scalars", c_vp), ("atom_draws", c_vp), ("code_u", c_vp),
                ("code_g", c_vp), ("workspace", c_vp), ("i_offset", c_i64), ("n_global", c_i64),
                ("allreduce", ALLREDUCE_FN), ("allreduce_ctx", c_vp), ("codes_zero", c_i32)]


PB_DRAW_PRIOR, PB_DRAW_EPOCH, PB_DRAW_POSTERIOR = 0, 1, 2
PB_INIT_PRIOR, PB_INIT_DATA = 0, 1
DRAW_FN = ctypes.CFUNCTYPE(c_i32, c_vp, c_i32, c_i64, ctypes.POINTER(c_i32), ctypes.POINTER(c_f64),
                           ctypes.POINTER(c_f64), ctypes.POINTER(c_f64), ctypes.POINTER(c_f64))


class ProblemDesc(ctypes.Structure):
    _fields_ = [("grid", GridDesc), ("num_atoms", c_i32), ("hyper", c_f64 * 6), ("seed", c_u64),
                ("mean_subtract", c_i32), ("epochs_per_frame", c_i32), ("freeze_dict", c_i32),
                ("data_consistency", c_i32), ("warm_start", c_i32), ("average_last", c_i32),
                ("replay", c_i32), ("init_mode", c_i32), ("draw", DRAW_FN), ("draw_ctx", c_vp)]


# name -> (restype, argtypes); exactly the functions include/pb200.h declares.
SIGNATURES = {
    "pb_last_error": (ctypes.c_char_p, []),
    "pb_version": (c_i32, []),
    "pb_device_count": (c_i32, []),
    "pb_grid_counts": (c_i32, [ctypes.POINTER(GridDesc), c_vp, c_vp, c_vp]),
    "pb_extract_patches": (c_i32, [ctypes.POINTER(GridDesc), c_vp, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp,
                                   c_vp, c_vp]),
    "pb_extract_patch_range": (c_i32, [ctypes.POINTER(GridDesc), c_vp, c_i32, c_vp, c_i32, c_i64, c_i64, c_vp,
                                       c_vp, c_vp, c_vp, c_vp]),
    "pb_reconstitute": (c_i32, [ctypes.POINTER(GridDesc), c_vp, c_f32, c_vp, c_vp, c_vp, c_i32, c_i32,
                                c_vp, c_vp, c_vp]),
    "pb_coverage_map": (c_i32, [ctypes.POINTER(GridDesc), c_vp, c_vp]),
    "pb_ola_partial": (c_i32, [ctypes.POINTER(GridDesc), c_vp, c_f32, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "pb_residual_full": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_i64, c_vp]),
    "pb_compose_estimates": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_i64, c_i32, c_vp]),
    "pb_atom_moments": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "pb_shift_atom": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "pb_code_moments": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "pb_shift_codes": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "pb_masked_sq_norm": (c_i32, [c_vp, c_i64, c_vp, c_vp, c_vp]),
    "pb_index_bytes": (ctypes.c_size_t, [c_i64, c_i32, c_i64]),
    "pb_build_index": (c_i32, [ctypes.POINTER(PatchIndex), c_vp, c_vp, c_vp, c_vp]),
    "pb_index_refresh_values": (c_i32, [ctypes.POINTER(PatchIndex), c_vp, c_vp, c_vp]),
    "pb_epoch_workspace_bytes": (ctypes.c_size_t, [c_i64, c_i32, c_i32, c_i64]),
    "pb_code_pitch": (c_i64, [c_i64]),
    "pb_gibbs_epoch": (c_i32, [ctypes.POINTER(EpochDesc), c_vp, c_vp]),
    "pb_phase_timing": (c_i32, [c_i32]),
    "pb_phase_read": (c_i32, [c_vp, c_vp]),
    "pb_dict_profile": (c_i32, [c_i32, c_vp]),
    "pb_problem_create": (c_i32, [ctypes.POINTER(ProblemDesc), ctypes.POINTER(c_vp)]),
    "pb_problem_destroy": (c_i32, [c_vp]),
    "pb_problem_submit_frame": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "pb_problem_submit_frame_ex": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pb_problem_residual_map": (c_i32, [c_vp, c_vp]),
    "pb_problem_adaptive_mask": (c_i32, [c_vp, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, c_i64, c_vp,
                                         ctypes.POINTER(c_i32)]),
    "pb_adaptive_mask": (c_i32, [c_vp, c_i64, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, c_i64, c_vp,
                                 ctypes.POINTER(c_i32), c_vp]),
    "pb_problem_install_dictionary": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32]),
    "pb_problem_transfer_dictionary": (c_i32, [c_vp, c_vp, c_i32]),
    "pb_normalize_observed": (c_i32, [c_vp, c_vp, c_i64, c_vp, ctypes.POINTER(c_f64), ctypes.POINTER(c_f64), c_vp]),
    "pb_transfer_atoms": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "pb_problem_render_atlas": (c_i32, [c_vp, c_vp]),
    "pb_atlas_shape": (c_i32, [c_i32, c_i32, c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "pb_render_atlas": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "pb_nccl_unique_id": (c_i32, [c_vp]),
    "pb_nccl_comm_create": (c_i32, [c_vp, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "pb_nccl_comm_destroy": (c_i32, [c_vp]),
    "pb_nccl_allreduce": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp]),
    "pb_problem_last_gpu_ms": (c_f32, [c_vp]),
    "pb_problem_get_dictionary": (c_i32, [c_vp, c_vp, c_vp, ctypes.POINTER(Scalars)]),
}

_lib = None


def load():
    """Load libpb200.so (raises if it has not been built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"pb200 CUDA library not built ({LIB_PATH}); run __graft_entry__.build() "
                "or `make -C paper_2311_15061_b200/csrc`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class PBError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"pb200 error {code}: {msg}")
        self.code = code


def check(rc: int, exc_map=None):
    if rc == PB_OK:
        return
    msg = load().pb_last_error().decode(errors="replace")
    if exc_map and rc in exc_map:
        raise exc_map[rc](msg)
    raise PBError(rc, msg)


def call(name, *args, exc_map=None):
    check(getattr(load(), name)(*args), exc_map)
