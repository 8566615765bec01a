"""Console-facing outputs of the live path (server.py:33-120): the dictionary
atlas rendered on the device from the device-resident atoms, and the uint8
wire frames (the panels themselves are produced on device by
``LiveProblem.submit_frame(..., panels=True)``).
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np

from . import _lib

FRAME_MASKED_INPUT = 0
FRAME_RECONSTRUCTION = 1
FRAME_DICT_ATLAS = 2
FRAME_GROUND_TRUTH = 3
DTYPE_U8 = 1
_HEADER = struct.Struct("<BBHIIII")   # server.py:38-39


def atlas_shape(num_atoms: int, patch_shape) -> tuple[int, int]:
    shape = (ctypes.c_int32 * 4)(*[int(b) for b in patch_shape])
    h, w = ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.check(_lib.load().pb_atlas_shape(int(num_atoms), len(patch_shape), shape, ctypes.byref(h),
                                          ctypes.byref(w)), {_lib.PB_EVALUE: ValueError})
    return int(h.value), int(w.value)


def render_dictionary_atlas(dictionary, as_uint8: bool = False) -> np.ndarray:
    """server.render_dictionary_atlas (server.py:84-120) on the device: atoms
    min-max normalised (constant atoms mid-grey), highest pi first (ties by
    index), ceil(sqrt(K)) grid with 1-pixel mid-grey separators."""
    import torch

    atoms = torch.as_tensor(np.asarray(dictionary.atoms) if not isinstance(dictionary.atoms, torch.Tensor)
                            else dictionary.atoms, dtype=torch.float32).to("cuda").contiguous()
    pi = torch.as_tensor(np.asarray(dictionary.pi) if not isinstance(dictionary.pi, torch.Tensor)
                         else dictionary.pi, dtype=torch.float64).to("cuda").contiguous()
    shape = tuple(int(b) for b in dictionary.patch_shape)
    h, w = atlas_shape(atoms.shape[0], shape)
    out = torch.empty((h, w), dtype=torch.uint8 if as_uint8 else torch.float64, device="cuda")
    cshape = (ctypes.c_int32 * 4)(*shape)
    _lib.check(_lib.load().pb_render_atlas(atoms.data_ptr(), pi.data_ptr(), atoms.shape[0], len(shape), cshape,
                                           None if as_uint8 else out.data_ptr(), out.data_ptr() if as_uint8 else None,
                                           torch.cuda.current_stream().cuda_stream), {_lib.PB_EVALUE: ValueError})
    return out.cpu().numpy()


def pack_wireframe(frame_type: int, problem_id: int, frame_id: int, panel: np.ndarray) -> bytes:
    """server.py:55-61: header + uint8 payload (panels are quantized on device)."""
    data = np.asarray(panel)
    if data.dtype != np.uint8:
        raise ValueError("wire panels are uint8 (quantize on device: LiveProblem.submit_frame(panels=True))")
    height, width = data.shape
    return _HEADER.pack(frame_type, DTYPE_U8, problem_id, width, height, frame_id, 0) + data.tobytes()


def unpack_wireframe(message: bytes) -> tuple[dict, np.ndarray]:
    """server.py:64-82."""
    if len(message) < _HEADER.size:
        raise ValueError("wire frame shorter than its header")
    ftype, dtype, problem_id, width, height, frame_id, reserved = _HEADER.unpack_from(message)
    if dtype != DTYPE_U8:
        raise ValueError(f"unknown wire dtype {dtype}")
    payload = message[_HEADER.size:]
    if len(payload) != width * height:
        raise ValueError(f"wire payload is {len(payload)} bytes, expected {width * height}")
    header = {"type": ftype, "problem_id": problem_id, "width": width, "height": height, "frame_id": frame_id,
              "reserved": reserved}
    return header, np.frombuffer(payload, dtype=np.uint8).reshape(height, width)
