"""Multi-GPU sharding of the Gibbs sweep.

One process per GPU.  The patch grid of one frame is cut into contiguous patch
ranges (rank r holds global patches [N*r/W, N*(r+1)/W)); the dictionary D, pi
and the precisions are replicated.  Exchanges per epoch:

* dictionary step — per block of 8 atoms, the 48*P per-pixel moment/Gram sums
  (f64) each rank accumulated over its own observed elements are allreduced,
  then every rank performs the same 8 sequential atom draws (draws keyed by
  global atom and pixel index) — bpfa.py:299-307 with the reduction split
  across ranks;
* code step — none: patches are independent; draws are keyed by the GLOBAL
  patch index, so a sharded run consumes exactly the 1-GPU draw streams;
* pi / gamma — the usage counts m_k and sum S^2, sum R^2 are allreduced, then
  every rank draws identical pi / gamma (bpfa.py:313-333);
* overlap-add — raw per-element sums of each shard (pb_ola_partial) are
  allreduced and divided by the analytic coverage.

Results equal the single-GPU run up to floating-point summation order.  The
collective is a small interface: `TorchCollective` uses torch.distributed
(NCCL on GPUs, gloo on CPU); `LocalCollective` lets W "ranks" run as threads
on one GPU for testing (sequential kernels, no cross-rank device waits).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib
from . import bpfa as _bpfa
from .patches import PatchMatrix, PatchSpec, ShapeError, _ptr, _stream, to_device

_DTYPES = {0: torch.float64, 1: torch.int32}


def shard_range(n: int, world: int, rank: int):
    """Global patch range [lo, hi) of `rank` (contiguous, sizes differ by <= 1)."""
    return n * rank // world, n * (rank + 1) // world


class Collective:
    world: int = 1
    rank: int = 0

    def allreduce_(self, t: torch.Tensor) -> None:
        raise NotImplementedError


class TorchCollective(Collective):
    """torch.distributed sum-allreduce on the default process group."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allreduce_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)


class NcclCollective(Collective):
    """A native NCCL communicator owned by the C library (pb_nccl_*): the
    sweep's exchanges are ncclAllReduce calls the library enqueues on the epoch
    stream itself (no host callback per exchange).  The 128-byte unique id is
    broadcast over torch.distributed (any backend); ``NcclCollective.single()``
    makes a one-rank communicator (tests)."""

    def __init__(self, group=None, _single=False):
        import torch

        torch.cuda.nccl.version()  # load the process's libnccl (the library dlopens the same copy)
        uid = (ctypes.c_uint8 * 128)()
        if _single:
            self.world, self.rank = 1, 0
            _lib.call("pb_nccl_unique_id", uid)
        else:
            import torch.distributed as dist

            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
            if self.rank == 0:
                _lib.call("pb_nccl_unique_id", uid)
            dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
            dist.broadcast(t, 0, group=group)
            uid = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        self.handle = ctypes.c_void_p()
        _lib.call("pb_nccl_comm_create", uid, self.world, self.rank, ctypes.byref(self.handle))

    @classmethod
    def single(cls):
        return cls(_single=True)

    def allreduce_(self, t):
        if not t.is_cuda:
            raise ValueError("NcclCollective reduces device tensors")
        dt = {torch.float64: 0, torch.int32: 1}[t.dtype]
        _lib.call("pb_nccl_allreduce", self.handle, t.data_ptr(), t.numel(), dt, torch.cuda.current_stream().cuda_stream)

    def close(self):
        if self.handle:
            _lib.call("pb_nccl_comm_destroy", self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class LocalCollective(Collective):
    """W ranks as host threads sharing one device (tests): a sum over the ranks'
    tensors in rank order, written back to every rank."""

    class _Hub:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, hub: "LocalCollective._Hub", rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    @classmethod
    def group(cls, world):
        hub = cls._Hub(world)
        return [cls(hub, r) for r in range(world)]

    def allreduce_(self, t):
        torch.cuda.current_stream().synchronize() if t.is_cuda else None
        self.hub.slots[self.rank] = t
        self.hub.barrier.wait()
        if self.rank == 0:
            acc = self.hub.slots[0].clone()
            for other in self.hub.slots[1:]:
                acc += other.to(acc.device)
            if acc.is_cuda:
                torch.cuda.current_stream().synchronize()
            self.hub.result = acc
        self.hub.barrier.wait()
        t.copy_(self.hub.result.to(t.device))
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        self.hub.barrier.wait()


class _CudaView:
    """Zero-copy torch view of a raw device buffer handed over the C ABI."""

    def __init__(self, ptr, count, dtype):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": {torch.float64: "<f8", torch.int32: "<i4"}[dtype],
                                         "data": (int(ptr), False), "version": 3}


def _callback(comm: Collective):
    def fn(ctx, ptr, count, dtype, stream):
        try:
            view = torch.as_tensor(_CudaView(ptr, count, _DTYPES[dtype]), device="cuda")
            comm.allreduce_(view)
            return 0
        except Exception:  # noqa: BLE001 — reported to C as a failure code
            import traceback

            traceback.print_exc()
            return 1

    return _lib.ALLREDUCE_FN(fn)


def extract_patch_shard(tensor, mask, spec: PatchSpec, mean_subtract: bool, comm: Collective) -> PatchMatrix:
    """This rank's contiguous share of extract_patches (patches.py:125-164)."""
    shape = tuple(int(m) for m in tensor.shape)
    spec.validate_for(shape)
    if tuple(mask.shape) != shape:
        raise ShapeError(f"mask shape {tuple(mask.shape)} != tensor shape {shape}")
    t = to_device(tensor, torch.float64)
    m = to_device(mask, torch.uint8) if not (isinstance(mask, torch.Tensor) and mask.dtype == torch.uint8) \
        else to_device(mask)
    n_global = spec.num_patches(shape)
    lo, hi = shard_range(n_global, comm.world, comm.rank)
    n, p = hi - lo, spec.patch_size
    values = torch.empty((p, n), dtype=torch.float32, device=t.device)
    obs = torch.empty((p, n), dtype=torch.uint8, device=t.device)
    means = torch.empty((n,), dtype=torch.float32, device=t.device)
    counts = torch.empty((n,), dtype=torch.int32, device=t.device)
    _lib.call("pb_extract_patch_range", ctypes.byref(spec.desc(shape)), _ptr(t), 1, _ptr(m), int(bool(mean_subtract)),
              lo, n, _ptr(values), _ptr(obs), _ptr(means), _ptr(counts), _stream())
    n_obs_local = counts.sum(dtype=torch.int64)
    tot = torch.stack([n_obs_local]).to(torch.float64)
    comm.allreduce_(tot)
    pm = PatchMatrix(values, obs, means, counts, shape, spec, bool(mean_subtract), int(n_obs_local.item()))
    pm.first_patch, pm.n_global, pm.n_obs_global = lo, n_global, int(round(float(tot.item())))
    return pm


def gibbs_epoch_sharded(state, pm: PatchMatrix, hp, comm: Collective, freeze_dict: bool = False,
                        check: bool = True):
    """One sharded sweep (device Philox draws); mutates and returns `state`."""
    _bpfa._check_state(state, pm)
    d, m = _bpfa._epoch_desc(state, pm, hp, freeze_dict, _lib.PB_RNG_PHILOX)
    d.i_offset = pm.first_patch
    d.n_global = pm.n_global
    d.n_obs = pm.n_obs_global
    if isinstance(comm, NcclCollective):  # native: ncclAllReduce enqueued by the library on the epoch stream
        cb = ctypes.cast(_lib.load().pb_nccl_allreduce, _lib.ALLREDUCE_FN)
        d.allreduce_ctx = comm.handle
    else:
        cb = _callback(comm)
    d.allreduce = cb
    _lib.call("pb_gibbs_epoch", ctypes.byref(d), _ptr(m), _stream())
    if check:
        s = state._sc()
        if s.diverged:
            raise _bpfa.DivergenceError(f"non-finite state at epoch {s.epoch}")
    return state


def infer_sharded(pm: PatchMatrix, hp, epochs: int, seed: int, comm: Collective, average_last: int = 1,
                  state=None):
    """bpfa.infer (bpfa.py:379-414) over a patch shard: (state, estimates of this shard)."""
    if epochs < 1:
        raise ValueError("epochs must be >= 1")
    if state is None:
        state = _bpfa.init_state(pm, hp, seed, init_mode="prior")
    average_last = max(1, min(int(average_last), epochs))
    tail = None
    for t in range(epochs):
        gibbs_epoch_sharded(state, pm, hp, comm, check=(t == epochs - 1))
        if t >= epochs - average_last:
            e = _bpfa.compose_estimates(state, out=tail, accumulate=tail is not None)
            tail = e.T
    return state, (tail / average_last).T if average_last > 1 else tail.T


def reconstitute_sharded(pm: PatchMatrix, estimates, comm: Collective, est_scale: float = 1.0) -> np.ndarray:
    """reconstitute (patches.py:188-215) from per-rank shard estimates: every rank
    gets the full f64 tensor."""
    e = estimates.T if estimates.shape[0] == pm.num_patches else estimates
    e = e.contiguous().to(torch.float32)
    acc = torch.zeros(pm.tensor_shape, dtype=torch.float64, device=e.device)
    g = pm.spec.desc(pm.tensor_shape)
    _lib.call("pb_ola_partial", ctypes.byref(g), _ptr(e), float(est_scale), _ptr(pm.means_dev), pm.first_patch,
              pm.num_patches, _ptr(acc), _stream())
    comm.allreduce_(acc)
    cov = torch.empty(pm.tensor_shape, dtype=torch.int32, device=e.device)
    _lib.call("pb_coverage_map", ctypes.byref(g), _ptr(cov), _stream())
    out = torch.where(cov > 0, acc / cov.clamp(min=1).to(torch.float64), torch.zeros_like(acc))
    return out.cpu().numpy()
