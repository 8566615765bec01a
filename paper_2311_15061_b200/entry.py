"""The reference's train / inpaint entry flows (patchbeam cli.py) as array-level
API calls on the device — the file I/O and argument parsing of the CLI stay out
of scope, the steps between them are the same:

* ``normalize_observed``  cli.py:195-212 ``_normalize_observed``, on the device
  (pb_normalize_observed);
* ``inpaint``             cli.py:247-274 ``cmd_inpaint``: normalize -> extract ->
  infer -> overlap-add -> data consistency (-> optional SADF dictionary out);
* ``learn``               cli.py:342-386 ``cmd_learn``: per image i a mask keyed by
  ``seed + i``, the images' patch matrices concatenated, ``infer``, the learned
  dictionary (-> optional SADF file).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .bpfa import Dictionary, GibbsState, Hyperparams, infer
from .patches import PatchMatrix, PatchSpec, ShapeError, _ptr, _stream, extract_patches, reconstitute, to_device


def normalize_observed(frame, mask):
    """cli.py:195-212: (frame mapped to [0, 1] from its observed values, scale,
    offset).  Identity (scale 1, offset 0) when the observed values already lie
    in [0, 1] or nothing is observed; a constant observed set maps the observed
    elements to 0 (scale 1, offset = that value).  Host arrays in -> host array
    out; CUDA tensors in -> CUDA tensor out."""
    dev_in = isinstance(frame, torch.Tensor) and frame.is_cuda
    f = to_device(frame, torch.float64)
    m = to_device(mask, torch.uint8) if not (isinstance(mask, torch.Tensor) and mask.dtype == torch.uint8) \
        else to_device(mask)
    if tuple(f.shape) != tuple(m.shape):
        raise ShapeError(f"mask shape {tuple(m.shape)} != frame shape {tuple(f.shape)}")
    out = torch.empty_like(f)
    scale, offset = ctypes.c_double(), ctypes.c_double()
    _lib.call("pb_normalize_observed", _ptr(f), _ptr(m), f.numel(), _ptr(out), ctypes.byref(scale),
              ctypes.byref(offset), _stream())
    return (out if dev_in else out.cpu().numpy()), float(scale.value), float(offset.value)


# the reference's private name (cli.py:195)
_normalize_observed = normalize_observed


@dataclass
class InpaintResult:
    reconstruction: np.ndarray      # in the normalized units of the frame (cli.py writes recon*scale + offset)
    state: GibbsState
    scale: float
    offset: float


def inpaint(frame, mask, patch_spec: PatchSpec, hyperparams: Hyperparams | None = None, epochs: int = 20,
            seed: int = 0, freeze_dict: bool = False, initial_dict: Dictionary | None = None,
            init_mode: str = "data", average_last: int = 1, mean_subtract: bool = True,
            data_consistency: bool = True, rng: str | None = None, dict_out: str | None = None) -> InpaintResult:
    """cmd_inpaint (cli.py:247-274) for arrays: the reference's inpaint flow."""
    hp = hyperparams or Hyperparams()
    m = np.asarray(mask, dtype=bool) if not isinstance(mask, torch.Tensor) else mask
    f, scale, offset = normalize_observed(frame, m)
    ms = bool(mean_subtract) and len(patch_spec.patch_shape) == 2        # cli.py:251
    pm = extract_patches(f, m, patch_spec, mean_subtract=ms)
    state, est = infer(pm, hp, epochs=epochs, seed=seed, freeze_dict=freeze_dict, initial_dict=initial_dict,
                       init_mode=init_mode, average_last=average_last, rng=rng)
    if data_consistency:                                                  # cli.py:264-265
        recon = reconstitute(pm, est, dc_original=f, dc_mask=m)
    else:
        recon = reconstitute(pm, est)
    if dict_out:
        from .formats import write_dict

        write_dict(dict_out, state.dictionary.to_host())
    return InpaintResult(recon, state, scale, offset)


def concat_patch_matrices(parts) -> PatchMatrix:
    """cli.py:371-379: one patch matrix of all images' patches (rows in image
    order; the first image's tensor shape and spec, as the reference keeps)."""
    if not parts:
        raise ValueError("no patch matrices")
    p = parts[0].patch_size
    if any(q.patch_size != p for q in parts):
        raise ShapeError("patch matrices of different patch sizes")
    values = torch.cat([q.values_pn for q in parts], dim=1).contiguous()
    obs = torch.cat([q.observed_pn for q in parts], dim=1).contiguous()
    means = torch.cat([q.means_dev for q in parts]).contiguous()
    counts = torch.cat([q.counts for q in parts]).contiguous()
    return PatchMatrix(values, obs, means, counts, parts[0].tensor_shape, parts[0].spec, parts[0].mean_subtracted,
                       sum(q.n_obs for q in parts))


@dataclass
class LearnResult:
    dictionary: Dictionary
    state: GibbsState
    num_patches: int


def learn(images, patch_spec: PatchSpec, num_atoms: int = 64, epochs: int = 20, seed: int = 0,
          mask_ratio: float = 0.2, mean_subtract: bool = True, rng: str | None = None,
          dict_out: str | None = None) -> LearnResult:
    """cmd_learn (cli.py:342-386) for arrays: per image i a uniform-random mask
    keyed by seed + i (SamplerSpec(ratio=mask_ratio, seed=seed + i)), the patch
    matrices concatenated, infer with the default (data) init, the dictionary."""
    from .inputs import make_mask

    if len(images) == 0:
        raise ValueError("no input images found")
    ms = bool(mean_subtract) and len(patch_spec.patch_shape) == 2
    parts = []
    for i, img in enumerate(images):
        shape = tuple(int(s) for s in img.shape)
        mask = make_mask(shape, mask_ratio, "uniform-random", seed + i)
        parts.append(extract_patches(img, mask, patch_spec, mean_subtract=ms))
    pm = concat_patch_matrices(parts)
    state, _ = infer(pm, Hyperparams(num_atoms=num_atoms), epochs=epochs, seed=seed, rng=rng)
    if dict_out:
        from .formats import write_dict

        write_dict(dict_out, state.dictionary.to_host())
    return LearnResult(state.dictionary, state, pm.num_patches)
