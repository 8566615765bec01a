"""Live inpainting of one problem on the device: the hot slice of
``Pipeline.submit_frame`` (pipeline.py:217-276) behind the C ABI's stateful
problem (``pb_problem_*``), with the device-resident tail of SURVEY §8f:

* warm start (codes re-burn each frame; dictionary, pi and the precisions carry
  over, pipeline.py:230-238), device Philox draws;
* overlap-add, optional data consistency, uint8 wire panels of the
  reconstruction and of the masked input (server.py:46-53), all on device;
* the residual map (recon − previous recon)² kept on device (pipeline.py:265-269)
  and the adaptive-residual sampler on it (sampling.py:184-207: exact exploit
  set, device-stream explore set).

Inputs and outputs are host NumPy arrays (the C ABI copies them).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bpfa import Dictionary, Hyperparams, transfer_dictionary
from .patches import PatchSpec, ShapeError

_VALUE = {_lib.PB_EVALUE: ValueError}


@dataclass
class LiveFrame:
    reconstruction: np.ndarray           # f64, after data consistency when enabled
    panel: np.ndarray | None             # uint8 wire panel of the reconstruction
    masked_panel: np.ndarray | None      # uint8 wire panel of frame * mask
    gpu_ms: float                        # device time of the frame's GPU work


class LiveProblem:
    """One live problem (ProblemConfig + ProblemHandle of pipeline.py:36-110)."""

    def __init__(self, shape, patch_spec: PatchSpec, hyperparams: Hyperparams | None = None, seed: int = 0,
                 epochs_per_frame: int = 2, freeze_dict: bool = False, data_consistency: bool = False,
                 warm_start: bool = True, average_last: int = 1, mean_subtract: bool | None = None,
                 init_mode: str = "data", rng: str = "philox"):
        """``rng="philox"``: device draws (the fast path).  ``rng="numpy"``: replay
        mode — the native problem consumes the reference's own keyed streams
        (rng.py:25-32; bpfa.py:121-122, 293-333), drawn on the host by a callback
        the library invokes once per epoch (plus once for the pi / gamma draws),
        so a frame reproduces Pipeline.submit_frame's draws exactly."""
        self.shape = tuple(int(m) for m in shape)
        patch_spec.validate_for(self.shape)
        hp = hyperparams or Hyperparams()
        if mean_subtract is None:  # pipeline.py:60-64: on for 2-D patches only
            mean_subtract = len(patch_spec.patch_shape) == 2
        d = _lib.ProblemDesc()
        d.grid = patch_spec.desc(self.shape)
        d.num_atoms = hp.num_atoms
        for j, v in enumerate((hp.concentration_a, hp.concentration_b, hp.weight_shape, hp.weight_rate,
                               hp.noise_shape, hp.noise_rate)):
            d.hyper[j] = v
        d.seed = int(seed)
        d.mean_subtract = int(bool(mean_subtract))
        d.epochs_per_frame = int(epochs_per_frame)
        d.freeze_dict = int(bool(freeze_dict))
        d.data_consistency = int(bool(data_consistency))
        d.warm_start = int(bool(warm_start))
        d.average_last = int(average_last)
        if init_mode not in ("data", "prior"):
            raise ValueError(f"unknown init mode {init_mode!r}")
        d.init_mode = _lib.PB_INIT_DATA if init_mode == "data" else _lib.PB_INIT_PRIOR
        self._draw = None
        if rng == "numpy":
            self._draw = _lib.DRAW_FN(_replay_provider(int(seed), hp, spec_n(patch_spec, self.shape),
                                                       patch_spec.patch_size))
            d.replay = 1
            d.draw = self._draw
        elif rng != "philox":
            raise ValueError(f"unknown rng mode {rng!r}")
        self._lib = _lib.load()
        self._h = ctypes.c_void_p()
        _lib.check(self._lib.pb_problem_create(ctypes.byref(d), ctypes.byref(self._h)))
        self.num_atoms, self.patch_size = hp.num_atoms, patch_spec.patch_size
        self.patch_shape = tuple(int(b) for b in patch_spec.patch_shape)
        rank = len(self.shape)
        self.panel_shape = self.shape[:2] if rank in (2, 3) else None
        self.frames_processed = 0

    def close(self):
        if self._h:
            self._lib.pb_problem_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def submit_frame(self, frame, mask, panels: bool = False) -> LiveFrame:
        frame = np.ascontiguousarray(frame, dtype=np.float64)
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        if frame.shape != self.shape or mask.shape != self.shape:
            raise ShapeError(f"frame {frame.shape} / mask {mask.shape} do not match the problem shape {self.shape}")
        out = np.empty(self.shape, dtype=np.float64)
        pnl = msk = None
        if panels:
            if self.panel_shape is None:
                raise ValueError(f"wire panels must be 2D, got rank {len(self.shape)}")
            pnl = np.empty(self.panel_shape, dtype=np.uint8)
            msk = np.empty(self.panel_shape, dtype=np.uint8)
        _lib.check(self._lib.pb_problem_submit_frame_ex(
            self._h, frame.ctypes.data, mask.ctypes.data, out.ctypes.data,
            pnl.ctypes.data if pnl is not None else None, msk.ctypes.data if msk is not None else None), _VALUE)
        self.frames_processed += 1
        return LiveFrame(out, pnl, msk, float(self._lib.pb_problem_last_gpu_ms(self._h)))

    def residual_map(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=np.float64)
        _lib.check(self._lib.pb_problem_residual_map(self._h, out.ctypes.data))
        return out

    def adaptive_mask(self, ratio: float, exploit_fraction: float = 0.5, seed: int = 0,
                      frame_index: int | None = None) -> np.ndarray:
        """The next mask from the device residual map (sampling.py:184-207)."""
        fi = self.frames_processed if frame_index is None else int(frame_index)
        out = np.empty(self.shape, dtype=np.uint8)
        status = ctypes.c_int32(0)
        _lib.check(self._lib.pb_problem_adaptive_mask(self._h, float(ratio), float(exploit_fraction), int(seed), fi,
                                                      out.ctypes.data, ctypes.byref(status)), _VALUE)
        return out.astype(bool)

    def install_dictionary(self, dictionary, freeze: bool | None = None) -> None:
        """Pipeline._install_dictionary (pipeline.py:145-167): the dictionary is
        reshaped to this problem's patch shape (bpfa.transfer_dictionary,
        bpfa.py:417-458, on device); codes reset; any atom count (the problem's
        K-dependent buffers are re-sized); pending until the first frame."""
        moved = transfer_dictionary(dictionary, self.patch_shape, self.shape)
        atoms = np.ascontiguousarray(_host(moved.atoms, np.float32))
        pi = np.ascontiguousarray(_host(moved.pi, np.float64))
        _lib.check(self._lib.pb_problem_install_dictionary(self._h, atoms.ctypes.data, pi.ctypes.data,
                                                           atoms.shape[0], -1 if freeze is None else int(bool(freeze))),
                   _VALUE)
        self.num_atoms = atoms.shape[0]

    def transfer_from(self, src: "LiveProblem", freeze: bool = False) -> None:
        """Pipeline.transfer_between(src, self) (pipeline.py:294-304), device to device."""
        transfer_between(src, self, freeze)

    def snapshot_dictionary(self) -> Dictionary:
        """Pipeline.snapshot_dictionary (pipeline.py:280-286), on the host."""
        atoms, pi, _ = self.dictionary()
        return Dictionary(atoms.astype(np.float64), pi, self.patch_shape)

    def render_atlas(self) -> np.ndarray:
        """The current dictionary atlas as a uint8 wire panel (server.py:84-120), on device."""
        from .display import atlas_shape

        out = np.empty(atlas_shape(self.num_atoms, self.patch_shape), dtype=np.uint8)
        _lib.check(self._lib.pb_problem_render_atlas(self._h, out.ctypes.data), _VALUE)
        return out

    def dictionary(self):
        atoms = np.empty((self.num_atoms, self.patch_size), dtype=np.float32)
        pi = np.empty(self.num_atoms, dtype=np.float64)
        sc = _lib.Scalars()
        _lib.check(self._lib.pb_problem_get_dictionary(self._h, atoms.ctypes.data, pi.ctypes.data, ctypes.byref(sc)))
        return atoms, pi, sc


def _host(x, dtype):
    import torch

    return (x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)).astype(dtype)


def transfer_between(src: LiveProblem, dst: LiveProblem, freeze: bool = False) -> None:
    """Pipeline.transfer_between (pipeline.py:294-304): install src's current
    dictionary into dst (reshaped by the transfer_dictionary rules on the device;
    dst codes reset; dst keeps its precisions and epoch counter)."""
    _lib.check(_lib.load().pb_problem_transfer_dictionary(src._h, dst._h, int(bool(freeze))),
               {_lib.PB_EVALUE: ValueError, _lib.PB_ESHAPE: ShapeError})
    dst.num_atoms = src.num_atoms


def spec_n(spec: PatchSpec, shape):
    return int(spec.num_patches(shape))


def _replay_provider(seed: int, hp: Hyperparams, n: int, p: int):
    """The reference's draws for the native replay mode (pb_draw_fn)."""
    import math
    import traceback

    from .bpfa import PRECISION_FLOOR
    from .rng import DOMAIN_ATOM, DOMAIN_CODE, DOMAIN_GAMMA, DOMAIN_INIT, DOMAIN_PI, keyed_rng

    k = hp.num_atoms

    def arr(ptr, shape):
        return np.ctypeslib.as_array(ptr, shape=shape)

    def fn(ctx, stage, epoch, m_counts, sums, out0, out1, out2):
        try:
            if stage == _lib.PB_DRAW_PRIOR:                     # bpfa.py:121-122
                a = arr(out0, (k, p))
                a[:] = keyed_rng(seed, DOMAIN_INIT).standard_normal((k, p)) / math.sqrt(p)
            elif stage == _lib.PB_DRAW_EPOCH:                   # bpfa.py:304, 258-259
                if out0:
                    a = arr(out0, (k, p))
                    for j in range(k):
                        keyed_rng(seed, DOMAIN_ATOM, epoch, j).standard_normal(out=a[j])
                u, g = arr(out1, (k, n)), arr(out2, (k, n))
                for j in range(k):
                    r = keyed_rng(seed, DOMAIN_CODE, epoch, j)
                    r.random(out=u[j])
                    r.standard_normal(out=g[j])
            elif stage == _lib.PB_DRAW_POSTERIOR:               # bpfa.py:313-333
                m = arr(m_counts, (k,)).astype(np.float64)
                sq_w, sq_r, n_obs = (float(x) for x in arr(sums, (3,)))
                sh_a = hp.concentration_a / k + m
                sh_b = hp.concentration_b * (k - 1) / k + n - m
                arr(out0, (k,))[:] = keyed_rng(seed, DOMAIN_PI, epoch).beta(
                    np.maximum(sh_a, PRECISION_FLOOR), np.maximum(sh_b, PRECISION_FLOOR))
                g5 = keyed_rng(seed, DOMAIN_GAMMA, epoch)
                gs = max(g5.gamma(hp.weight_shape + 0.5 * n * k, 1.0 / (hp.weight_rate + 0.5 * sq_w)),
                         PRECISION_FLOOR)
                ge = max(g5.gamma(hp.noise_shape + 0.5 * n_obs, 1.0 / (hp.noise_rate + 0.5 * sq_r)),
                         PRECISION_FLOOR)
                arr(out1, (2,))[:] = (gs, ge)
            else:
                return 1
            return 0
        except Exception:  # noqa: BLE001 — reported to C as a failure code
            traceback.print_exc()
            return 1

    return fn


def adaptive_mask(residual, ratio: float, exploit_fraction: float = 0.5, seed: int = 0, frame_index: int = 0):
    """sampling.py:184-207 on device for a residual map (host or CUDA tensor);
    returns (mask bool ndarray, all_zero flag)."""
    import torch

    r = torch.as_tensor(np.asarray(residual, dtype=np.float64) if not isinstance(residual, torch.Tensor)
                        else residual, dtype=torch.float64).to("cuda").contiguous()
    out = torch.empty(r.shape, dtype=torch.uint8, device="cuda")
    status = ctypes.c_int32(0)
    _lib.check(_lib.load().pb_adaptive_mask(r.data_ptr(), r.numel(), float(ratio), float(exploit_fraction), int(seed),
                                            int(frame_index), out.data_ptr(), ctypes.byref(status),
                                            torch.cuda.current_stream().cuda_stream), _VALUE)
    return out.cpu().numpy().astype(bool), bool(status.value)
