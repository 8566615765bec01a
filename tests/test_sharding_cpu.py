"""World-size-2 gloo test (CPU) of the sharding decomposition used by
paper_2311_15061_b200.parallel: patches split into contiguous global ranges,
dictionary moments summed across ranks before the (identical) atom draws,
code draws sliced by GLOBAL patch index from the reference streams, usage
counts / sum S^2 / sum R^2 allreduced before the pi / gamma draws, overlap-add
sums allreduced.  Run with the oracle's f64 kernels per shard, the sharded
epoch must reproduce the unsharded oracle epoch to 1e-12 (summation order)."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import _ckernels as ck
from oracle import bpfa as ob
from oracle import patches as op
from oracle.rng import DOMAIN_ATOM, DOMAIN_CODE, DOMAIN_GAMMA, DOMAIN_PI, keyed_rng
from paper_2311_15061_b200 import inputs
from paper_2311_15061_b200.parallel import TorchCollective, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sharded_epoch(st, pm_vals, pm_obs, hp, n_global, n_obs_global, lo, comm):
    """One epoch over the local shard rows [lo, lo+n) with cross-rank sums."""
    n, p = pm_vals.shape
    k_len = st.atoms.shape[0]
    epoch = st.epoch + 1

    class _PM:  # shard view for the oracle helpers
        values, observed = pm_vals, pm_obs

    r = ob.residual(_PM, st)
    for k in range(k_len):
        w = ob.active_weights(st, k)
        a, c = ck.atom_moments(r, pm_obs, w)
        ac = torch.from_numpy(np.concatenate([a, c]))
        comm.allreduce_(ac)
        a, c = ac[:p].numpy(), ac[p:].numpy()
        lam, mu = ob.atom_params(a, c, st.atoms[k], st.gamma_eps, float(p))
        new = mu + keyed_rng(st.seed, DOMAIN_ATOM, epoch, k).standard_normal(p) / np.sqrt(lam)
        ck.shift_atom(r, pm_obs, w, st.atoms[k] - new)
        st.atoms[k] = new
    for k in range(k_len):
        g = keyed_rng(st.seed, DOMAIN_CODE, epoch, k)
        u_all = g.random(n_global)
        g_all = g.standard_normal(n_global)
        ob.sample_codes(r, _PM, st, k, u_all[lo:lo + n], g_all[lo:lo + n])
    stats = torch.from_numpy(np.concatenate([st.usage.sum(axis=0).astype(np.float64),
                                             [float((st.weights * st.weights).sum()), ck.masked_sq_norm(r)]]))
    comm.allreduce_(stats)
    m, sw, sr = stats[:k_len].numpy(), float(stats[k_len]), float(stats[k_len + 1])
    sh_a = hp.concentration_a / k_len + m
    sh_b = hp.concentration_b * (k_len - 1) / k_len + n_global - m
    st.pi = keyed_rng(st.seed, DOMAIN_PI, epoch).beta(np.maximum(sh_a, 1e-12), np.maximum(sh_b, 1e-12))
    g5 = keyed_rng(st.seed, DOMAIN_GAMMA, epoch)
    st.gamma_s = max(g5.gamma(hp.weight_shape + 0.5 * n_global * k_len, 1.0 / (hp.weight_rate + 0.5 * sw)), 1e-12)
    st.gamma_eps = max(g5.gamma(hp.noise_shape + 0.5 * n_obs_global, 1.0 / (hp.noise_rate + 0.5 * sr)), 1e-12)
    st.epoch = epoch
    return st


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchCollective()
        img = inputs.synthetic_texture((30, 34), seed=2)
        mask = inputs.make_mask(img.shape, 0.3, "uniform-random", 2)
        full = op.extract_patches(img, mask, (5, 5), (), True)
        n_global = full.values.shape[0]
        lo, hi = shard_range(n_global, world, rank)
        vals, obs = full.values[lo:hi].copy(), full.observed[lo:hi].copy()
        hp = ob.Hyper(num_atoms=6)
        st0 = ob.init_state(full, hp, 9, "prior")
        st = ob.State(st0.atoms.copy(), st0.pi.copy(), st0.usage[lo:hi].copy(), st0.weights[lo:hi].copy(),
                      st0.gamma_s, st0.gamma_eps, 0, 9)
        for _ in range(3):
            _sharded_epoch(st, vals, obs, hp, n_global, int(full.observed.sum()), lo, comm)
        est = ob.compose_estimates(st)
        # sharded overlap-add: raw sums of own patches, allreduced, / coverage
        acc = np.zeros(int(np.prod(img.shape)))
        fi = op.flat_index(img.shape, (5, 5), (1, 1))[lo:hi]
        np.add.at(acc, fi.ravel(), (est + full.means[lo:hi, None]).ravel())
        acc_t = torch.from_numpy(acc)
        comm.allreduce_(acc_t)
        cov = op.coverage(img.shape, (5, 5), (1, 1)).ravel()
        rec = np.where(cov > 0, acc_t.numpy() / np.maximum(cov, 1), 0.0).reshape(img.shape)
        result_q.put((rank, lo, st.atoms, st.usage, st.weights, st.pi, st.gamma_s, st.gamma_eps, rec))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_epoch_matches_oracle():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in procs]
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)

    img = inputs.synthetic_texture((30, 34), seed=2)
    mask = inputs.make_mask(img.shape, 0.3, "uniform-random", 2)
    full = op.extract_patches(img, mask, (5, 5), (), True)
    hp = ob.Hyper(num_atoms=6)
    st = ob.init_state(full, hp, 9, "prior")
    for _ in range(3):
        ob.gibbs_epoch(st, full, hp)
    rec_ref = op.reconstitute(full, ob.compose_estimates(st))

    for r in res:
        assert np.allclose(r[2], st.atoms, rtol=0, atol=1e-9), "replicated dictionary"
        assert np.allclose(r[5], st.pi, atol=1e-9)
        assert math.isclose(r[6], st.gamma_s, rel_tol=1e-9) and math.isclose(r[7], st.gamma_eps, rel_tol=1e-9)
        assert np.allclose(r[8], rec_ref, atol=1e-9), "sharded overlap-add"
    usage = np.concatenate([r[3] for r in res])
    weights = np.concatenate([r[4] for r in res])
    assert np.array_equal(usage, st.usage)
    assert np.allclose(weights, st.weights, atol=1e-9)
