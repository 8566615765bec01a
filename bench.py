#!/usr/bin/env python
"""Benchmark of the B200 BPFA Gibbs-sampling inpainting hot path.

Contract (see DESIGN.md §5/§6):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload: at N = 1 BASELINE.json configs[1] — 2-D 1024x1024 synthetic STEM-like
frame, 10% uniform sampling, 10x10 patches (stride 1, N = 1,030,225), K = 256
atoms.  At N > 1 configs[4] — a 4096x4096 frame, 10%, 8x8, K = 256 — cut into N
contiguous patch shards (strong scaling; configs[4] at N = 1 through the same
sharded code path is the base point under ``configs``).  One STEP = one full
Gibbs sweep (bpfa.gibbs_epoch: residual, dictionary step, code step, pi/gamma
draws) over the whole frame = N*K patch-atom updates.  Metric: patch-atom
updates/s (higher is better).

* value      device-resident throughput (state in HBM, CUDA events, max over ranks);
* e2e        one cold inpaint of the frame (50 / 10 epochs) per step through the C ABI
             with HOST buffers (pb_problem_submit_frame: H2D frame+mask, extract,
             sweeps, compose, overlap-add, D2H reconstruction);
* live       BASELINE configs[2]: 512x512 line-hop 25% frames, 8x8, K=256,
             2 warm-started epochs per frame, frames/s through the same C ABI;
* quality    PSNR / SSIM of the device result against the REFERENCE's on identical
             inputs and seeds (tests/golden/quality.json, produced by running
             patchbeam itself): replay mode (same draws) and Philox mode (mean
             over 3 seeds) for configs[0] in full, configs[2] live, a configs[1] crop;
* roofline   the dominant kernel (by measured phase time) against MEASURED_PEAKS.json;
* cpu_baseline  the reference's own CPU path — the unmodified patchbeam installed in
             baseline/_ref (its Numba kernels through bpfa.gibbs_epoch, all host
             threads) when present, else the oracle port (numpy + OpenMP C
             restatement, f64; measured 12 % slower than patchbeam on the box,
             profiles/r02/cpu_ref_vs_port.json) — on bounded bands of the same frame.

--impl reference runs that CPU path alone on the same metric and config (rank 0
only): each step is one full Gibbs epoch over one 64-row band of the frame,
consecutive steps walking the bands.

N GPUs: if WORLD_SIZE is unset, bench.py relaunches itself under
torch.distributed.run with N ranks.  The dictionary step's per-block moment sums
and the epoch statistics are allreduced by native NCCL calls the library
enqueues on the sweep's stream (parallel.NcclCollective).
"""

from __future__ import annotations

import argparse
import glob
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (configs[3]/[4] state no epoch count: 10 is assumed)
CFGS = {
    0: dict(shape=(256, 256), ratio=0.25, kind="uniform-random", patch=(8, 8), k=64, epochs=10, seed=0,
            what="2D 256x256 STEM-like, 25% uniform, 8x8, K=64, 10 iterations"),
    1: dict(shape=(1024, 1024), ratio=0.10, kind="uniform-random", patch=(10, 10), k=256, epochs=50, seed=0,
            what="configs[1] 1024x1024 STEM-like, 10% uniform, 10x10, K=256; step = 1 Gibbs sweep"),
    2: dict(shape=(512, 512), ratio=0.25, kind="line-hop", patch=(8, 8), k=256, epochs=2, seed=0,
            what="512x512 live frame, 25% line-hop, 8x8, K=256 (sweep rate; frames/s under 'live')"),
    3: dict(shape=(256, 256, 128), ratio=0.20, kind="uniform-random", patch=(8, 8, 4), k=512, epochs=10, seed=0,
            what="hyperspectral cube 256x256x128, 20% uniform, 8x8x4 patches, K=512, mean subtraction off"),
    4: dict(shape=(4096, 4096), ratio=0.10, kind="uniform-random", patch=(8, 8), k=256, epochs=10, seed=0,
            what="configs[4] 4096x4096 STEM-like, 10% uniform, 8x8, K=256, patch shards; step = 1 Gibbs sweep"),
}
CFG = CFGS[1]
LIVE = CFGS[2]
OTHER_CFGS = {c: CFGS[c] for c in (0, 2, 3, 4)}
CROP_ROWS = 64  # bounded CPU sample: 64-row bands of the frame


def workload(world):
    """The headline workload: configs[1] on one GPU, configs[4] patch-sharded on N > 1."""
    return CFGS[1] if world == 1 else CFGS[4]


def workload_inputs(cfg):
    from paper_2311_15061_b200 import inputs

    img = inputs.stem_lattice(cfg["shape"], seed=cfg["seed"])
    mask = inputs.make_mask(cfg["shape"], cfg["ratio"], cfg["kind"], cfg["seed"])
    return img, mask


def grid_n(shape, patch):
    return int(np.prod([m - b + 1 for m, b in zip(shape, patch)]))


# --------------------------------------------------------------------------- CPU
def cpu_epoch_sample(cfg, seconds_budget=20.0, steps=None, warmup=0):
    """Oracle (reference restatement) epochs on CROP_ROWS-row bands of the frame:
    step t runs one full Gibbs epoch over band t mod (rows / CROP_ROWS), so
    consecutive steps walk the whole frame; band setup is outside the timing."""
    from oracle import bpfa as ob
    from oracle import patches as op
    from oracle import _ckernels

    img, mask = workload_inputs(cfg)
    nbands = cfg["shape"][0] // CROP_ROWS
    hp = ob.Hyper(num_atoms=cfg["k"])

    def band(t):
        b = t % nbands
        sl = slice(b * CROP_ROWS, (b + 1) * CROP_ROWS)
        opm = op.extract_patches(np.ascontiguousarray(img[sl]), np.ascontiguousarray(mask[sl]), cfg["patch"], (),
                                 True)
        return opm, ob.init_state(opm, hp, cfg["seed"], "prior")

    for _ in range(warmup):
        opm, st = band(0)
        ob.gibbs_epoch(st, opm, hp)
    times, upd = [], 0
    t_all = time.perf_counter()
    t = 0
    while True:
        opm, st = band(t)
        t0 = time.perf_counter()
        ob.gibbs_epoch(st, opm, hp)
        times.append(time.perf_counter() - t0)
        upd += opm.values.shape[0] * cfg["k"]
        t += 1
        if steps is not None:
            if len(times) >= steps:
                break
        elif time.perf_counter() - t_all >= seconds_budget:
            break
    n_band = op.extract_patches(img[:CROP_ROWS], mask[:CROP_ROWS], cfg["patch"], (), False).values.shape[0]
    return dict(updates=upd, times=times, cores=_ckernels.num_threads(),
                sample=f"{len(times)} full Gibbs epoch(s) (K={cfg['k']}, f64, oracle port: numpy + OpenMP C "
                       f"kernels), each over one {CROP_ROWS}-row band of the frame (N={n_band}), consecutive "
                       f"epochs walking its {nbands} bands")


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available():
    return os.path.isdir(os.path.join(REF_DIR, "patchbeam"))


def ref_epoch_sample(cfg, seconds_budget=20.0, steps=None, warmup=1):
    """The UNMODIFIED reference (patchbeam from baseline/_ref, its own Numba kernels
    and public API, all host threads) on the same CROP_ROWS-row bands as
    cpu_epoch_sample.  The first warm-up epoch includes Numba's compilation."""
    import tempfile

    cache = os.path.join(ROOT, "baseline", "_numba_cache")   # git-ignored; compiled once per box
    try:
        os.makedirs(cache, exist_ok=True)
    except OSError:
        cache = tempfile.mkdtemp(prefix="numba_")
    os.environ.setdefault("NUMBA_CACHE_DIR", cache)
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import numba
    from patchbeam import bpfa as rb
    from patchbeam.patches import PatchSpec as RSpec
    from patchbeam.patches import extract_patches as rextract

    img, mask = workload_inputs(cfg)
    nbands = cfg["shape"][0] // CROP_ROWS
    hp = rb.Hyperparams(num_atoms=cfg["k"])

    def band(t):
        b = t % nbands
        sl = slice(b * CROP_ROWS, (b + 1) * CROP_ROWS)
        pm = rextract(np.ascontiguousarray(img[sl]), np.ascontiguousarray(mask[sl]), RSpec(cfg["patch"]),
                      mean_subtract=True)
        return pm, rb.init_state(pm, hp, cfg["seed"], init_mode="prior")

    for _ in range(max(1, warmup)):
        pm, st = band(0)
        rb.gibbs_epoch(st, pm, hp)
    times, upd = [], 0
    t_all = time.perf_counter()
    t = 0
    while True:
        pm, st = band(t)
        t0 = time.perf_counter()
        rb.gibbs_epoch(st, pm, hp)
        times.append(time.perf_counter() - t0)
        upd += pm.values.shape[0] * cfg["k"]
        t += 1
        if steps is not None:
            if len(times) >= steps:
                break
        elif time.perf_counter() - t_all >= seconds_budget:
            break
    return dict(updates=upd, times=times, cores=numba.get_num_threads(), kind="reference",
                sample=f"{len(times)} full Gibbs epoch(s) (K={cfg['k']}, f64) of the unmodified reference "
                       f"(patchbeam from baseline/_ref, Numba kernels, bpfa.gibbs_epoch), each over one "
                       f"{CROP_ROWS}-row band of the frame (N={pm.values.shape[0]}), consecutive epochs walking "
                       f"its {nbands} bands")


def cpu_reference_sample(cfg, **kw):
    """The reference's own CPU path when it is installed (baseline/_ref), else the
    oracle port of it (kind "port")."""
    if reference_available():
        try:
            return ref_epoch_sample(cfg, **kw)
        except Exception as e:  # noqa: BLE001 - fall back to the port, saying why
            r = cpu_epoch_sample(cfg, **kw)
            r["kind"] = "port"
            r["sample"] += f" (reference unavailable: {type(e).__name__}: {e})"
            return r
    r = cpu_epoch_sample(cfg, **kw)
    r["kind"] = "port"
    return r


def headline_config(world, n_units, extra=None):
    cfg = workload(world)
    c = {"workload": cfg["what"], "global_batch": n_units, "seq_len": 1,
         "parallelism": f"patch-shards{world}" if world > 1 else "single"}
    c.update(extra or {})
    return c


def run_reference_arm(args):
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cfg = workload(world)
    r = cpu_reference_sample(cfg, steps=args.steps, warmup=args.warmup)
    total = sum(r["times"])
    v = r["updates"] / total
    n_units = grid_n(cfg["shape"], cfg["patch"])
    line = {
        "impl": "reference", "metric": "BPFA patch-atom updates/sec", "value": v, "unit": "updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(r["times"]), "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": headline_config(world, n_units),
        "cpu_baseline": {"value": v, "unit": "updates/s", "cores": r["cores"], "kind": r["kind"],
                         "sample": r["sample"]},
        "e2e": {"value": v, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []          # (monotonic time, csv line)
        self.window = None       # (t0, t1) of the timed region

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window:
            t0, t1 = self.window
            inside = [x for x in lines if t0 <= x[0] <= t1 + 0.03]
            if not inside and lines:  # region shorter than the sampling period: nearest sample
                inside = [min(lines, key=lambda x: abs(x[0] - 0.5 * (t0 + t1)))]
            lines = inside
        for _, ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} runs with WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def relaunch_distributed(args):
    """`bench.py --gpus N` (N > 1) started without a launcher: re-exec under
    torch.distributed.run with N ranks on this node (rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def problem_desc(cfg, epochs, warm, dc):
    from paper_2311_15061_b200 import _lib
    from paper_2311_15061_b200.patches import PatchSpec

    d = _lib.ProblemDesc()
    d.grid = PatchSpec(cfg["patch"]).desc(cfg["shape"])
    d.num_atoms = cfg["k"]
    for j, v in enumerate((1.0, 1.0, 1e-6, 1e-6, 1e-6, 1e-6)):
        d.hyper[j] = v
    d.seed = cfg["seed"]
    d.mean_subtract = 1
    d.epochs_per_frame = epochs
    d.freeze_dict = 0
    d.data_consistency = int(dc)
    d.warm_start = int(warm)
    d.average_last = 1
    return d


FP32_PEAK_TF = 74.45  # derived: 148 SM x 128 lanes x 2 x 1.965 GHz


def config_inputs(cfg, seed=0):
    from paper_2311_15061_b200 import inputs

    if len(cfg["shape"]) == 2:
        img = inputs.stem_lattice(cfg["shape"], seed=seed)
    else:  # cube: a STEM-like band image with a smooth spectral modulation per band
        base = inputs.stem_lattice(cfg["shape"][:2], seed=seed)
        spec = 0.5 + 0.5 * np.sin(np.linspace(0.0, 3.0 * np.pi, cfg["shape"][2]))
        img = base[:, :, None] * spec[None, None, :]
    mask = inputs.make_mask(cfg["shape"], cfg["ratio"], cfg["kind"], seed)
    return img, mask


def all_configs(args):
    """Device sweep throughput of every other BASELINE config (same code path as
    `value`: state resident, CUDA events, philox draws), with the sweep's
    roofline: floor = max(12*|Omega|*K flops / FP32 peak, 15 B per update / HBM)."""
    import torch

    from paper_2311_15061_b200 import _lib
    from paper_2311_15061_b200 import bpfa as gb
    from paper_2311_15061_b200 import patches as pp
    from paper_2311_15061_b200.metrics import psnr

    lib = _lib.load()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    out = {}
    for cid, cfg in OTHER_CFGS.items():
        img, mask = config_inputs(cfg)
        pm = pp.extract_patches(img, mask, pp.PatchSpec(cfg["patch"]), len(cfg["shape"]) == 2)
        hp = gb.Hyperparams(num_atoms=cfg["k"])
        st = gb.init_state(pm, hp, 0, "prior")
        for _ in range(3):
            gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
        torch.cuda.synchronize()
        lib.pb_phase_timing(1)
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.config_steps):
            gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.config_steps
        phase = (ctypes.c_double * 4)()
        nph = ctypes.c_int64()
        lib.pb_phase_read(phase, ctypes.byref(nph))
        lib.pb_phase_timing(0)
        n, k = pm.num_patches, cfg["k"]
        upd = n * k
        floor_ms = 1e3 * max(12.0 * pm.n_obs * k / (FP32_PEAK_TF * 1e12), 15.0 * upd / (peaks["hbm_gbs"] * 1e9))
        est = gb.compose_estimates(st)
        rec = pp.reconstitute(pm, est)
        out[f"configs[{cid}]"] = {
            "workload": cfg["what"], "patches": n, "atoms": k, "patch_size": pm.patch_size,
            "observed_per_patch": pm.n_obs / n, "ms_per_sweep": ms, "updates_per_s": upd / (ms * 1e-3),
            "ms_per_run": ms * cfg["epochs"], "epochs_per_run": cfg["epochs"],
            "dict_ms": phase[1] / max(1, nph.value), "code_ms": phase[2] / max(1, nph.value),
            "roofline_floor_ms": floor_ms, "roofline_frac": floor_ms / ms,
            "psnr_db_after": psnr(rec, img), "sweeps": 3 + args.config_steps,
        }
        if st._sc().diverged:
            out[f"configs[{cid}]"]["diverged"] = True
        del st, pm, est, rec
        torch.cuda.empty_cache()
        if cid == 4:   # the N = 1 point of the N > 1 (patch-sharded, split-mode) code path
            out["configs[4]"]["sharded_1rank"] = sharded_point(args, cfg, img, mask)
            torch.cuda.empty_cache()
    return out


def sharded_point(args, cfg, img, mask):
    """configs[4] through the sharded code path with a one-rank NCCL communicator
    (split-mode dictionary step: per 8-atom block a pass, an ncclAllReduce of the
    moment sums and the atom update) — the base point of the N > 1 curve."""
    import torch

    from paper_2311_15061_b200 import bpfa as gb
    from paper_2311_15061_b200 import parallel as par
    from paper_2311_15061_b200 import patches as pp

    comm = par.NcclCollective.single()
    try:
        pm = par.extract_patch_shard(img, mask, pp.PatchSpec(cfg["patch"]), True, comm)
        hp = gb.Hyperparams(num_atoms=cfg["k"])
        st = gb.init_state(pm, hp, 0, "prior")
        for _ in range(3):
            par.gibbs_epoch_sharded(st, pm, hp, comm, check=False)
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.config_steps):
            par.gibbs_epoch_sharded(st, pm, hp, comm, check=False)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.config_steps
        return {"ms_per_sweep": ms, "updates_per_s": pm.n_global * cfg["k"] / (ms * 1e-3),
                "path": "parallel.gibbs_epoch_sharded, NcclCollective world 1 (split mode)"}
    finally:
        comm.close()


def quality_block():
    """Device PSNR / SSIM next to the REFERENCE's on identical inputs and seeds
    (tests/golden/quality.json, produced by patchbeam itself): replay mode of
    seed 0 (the reference's own draws) and the Philox-mode mean over seeds 0-2."""
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from quality_cases import SEEDS, reference_summary, run_device

    qref = json.load(open(os.path.join(ROOT, "tests", "golden", "quality.json")))
    out = {}
    for name, label in (("cfg0", "configs[0]"), ("cfg2", "configs[2] live, 3 frames"), ("cfg1crop", "configs[1] crop")):
        p_ref, s_ref = reference_summary(qref, name)
        rep = np.array(run_device(name, SEEDS[0], rng="numpy"))
        phi = np.array([run_device(name, sd, rng="philox") for sd in SEEDS])
        out[label] = {"ref_psnr": round(float(p_ref.mean()), 4), "ref_ssim": round(float(s_ref.mean()), 5),
                      "philox_psnr": round(float(phi[..., 0].mean()), 4),
                      "philox_ssim": round(float(phi[..., 1].mean()), 5),
                      "replay_dpsnr_max": float(np.abs(rep[:, 0] - p_ref[0]).max()),
                      "replay_dssim_max": float(np.abs(rep[:, 1] - s_ref[0]).max())}
    out["tolerance"] = "replay +-0.05 dB / +-0.001; philox mean over seeds 0-2 +-0.1 dB / +-0.002"
    return out


def run_gpu_arm(args):
    import torch

    from paper_2311_15061_b200 import _lib
    from paper_2311_15061_b200 import bpfa as gb
    from paper_2311_15061_b200 import patches as pp
    from paper_2311_15061_b200.metrics import psnr

    world, rank, local = dist_setup(args)
    lib = _lib.load()
    cfg = workload(world)
    img, mask = workload_inputs(cfg)
    hp = gb.Hyperparams(num_atoms=cfg["k"])
    comm = None
    if world > 1:
        # configs[4] in contiguous patch-range shards (strong scaling), D replicated;
        # the 44*P moment sums of each 8-atom block and the epoch statistics are
        # allreduced by native NCCL calls the library enqueues on the epoch stream
        from paper_2311_15061_b200 import parallel as par

        try:
            comm = par.NcclCollective()
        except Exception:  # noqa: BLE001 — no native NCCL: torch.distributed callback
            comm = par.TorchCollective()
        pm = par.extract_patch_shard(img, mask, pp.PatchSpec(cfg["patch"]), True, comm)
        sweep = lambda st: par.gibbs_epoch_sharded(st, pm, hp, comm, check=False)  # noqa: E731
        n_units = pm.n_global
    else:
        pm = pp.extract_patches(img, mask, pp.PatchSpec(cfg["patch"]), True)
        sweep = lambda st: gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)  # noqa: E731
        n_units = pm.num_patches
    n, k, p = pm.num_patches, cfg["k"], pm.patch_size
    split_code = pm.index().split_count > 0   # two code-step launches per sweep
    st = gb.init_state(pm, hp, cfg["seed"], "prior")
    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        sweep(st)
    torch.cuda.synchronize()
    lib.pb_phase_timing(1)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    t_start = time.monotonic()
    e0.record(stream)
    for _ in range(args.steps):
        sweep(st)
    e1.record(stream)
    torch.cuda.synchronize()
    clk.mark(t_start, time.monotonic())
    time.sleep(0.06)
    clk.__exit__(None, None, None)
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    phase = (ctypes.c_double * 4)()
    nph = ctypes.c_int64()
    lib.pb_phase_read(phase, ctypes.byref(nph))
    lib.pb_phase_timing(0)
    if st._sc().diverged:
        raise SystemExit("diverged")
    value = n_units * k * args.steps / (ms * 1e-3)   # whole-job updates/s (the frame's N*K per sweep)
    replicas = replica_check(st, world) if world > 1 else None

    # --- roofline of the dominant kernel ------------------------------------
    # the dictionary step runs k_dict_ell2 (two tile stages) whenever its shared memory fits (P <= 256),
    # else the single-stage k_dict_gram
    names = ["k_resid_compact (residual / carry)",
             ("k_dict_ell2" if p <= 256 else "k_dict_gram") + " (dictionary step)", "k_code_compact (code step)",
             "k_finish_stats+k_draw_pi_gamma"]
    per = [phase[i] / max(1, nph.value) for i in range(4)]
    dom = int(np.argmax(per))
    obs_per_patch = pm.n_obs / n
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "_fallback": True}
    # algorithmic bytes per patch-atom update for the dominant kernel
    if dom == 2:      # code step: read z,s + write z,s = 10 B / update, + R in (4|Omega|/K)
        alg_bytes = n * k * 10.0 + 4.0 * pm.n_obs
        alg_flops = n * k * 6.0 * obs_per_patch
    elif dom == 1:    # dictionary step: read z,s = 5 B / update + R in/out once
        alg_bytes = n * k * 5.0 + 8.0 * pm.n_obs
        alg_flops = n * k * 6.0 * obs_per_patch
    else:
        alg_bytes = n * k * 5.0 + 8.0 * pm.n_obs
        alg_flops = n * k * 2.0 * p
    dur_s = per[dom] * 1e-3
    achieved = alg_bytes / dur_s / 1e9
    # DRAM traffic per launch of the same kernel from the committed `ncu --set full`
    # capture (profiles/rNN/ncu_traffic.json, configs[1] sizes); null if absent
    traffic, traffic_src = None, None
    kname = names[dom].split()[0]
    for tf in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_traffic.json")), reverse=True):
        tj = json.load(open(tf))
        if kname in tj:
            traffic = tj[kname]["traffic_bytes"]
            traffic_src = os.path.relpath(tf, ROOT) + " @ " + tj.get("_capture", {}).get("commit", "?")
            break
    fp32_peak, fp32_src = FP32_PEAK_TF, "derived 148x128x2x1.965 GHz"
    if "fp32_tflops" in peaks:
        fp32_peak, fp32_src = float(peaks["fp32_tflops"]), "MEASURED_PEAKS.json fp32_tflops"
    else:
        for ff in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "fp32_peak.json")), reverse=True):
            fp32_peak = float(json.load(open(ff))["ffma2_tflops"])
            fp32_src = os.path.relpath(ff, ROOT) + " (tools/micro/ffma2_bench.cu on this pool's B200)"
            break
    roofline = {"bound": "hbm", "kernel": names[dom], "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "traffic_source": traffic_src,
                "peak_source": "fallback" if peaks.get("_fallback") else "MEASURED_PEAKS.json hbm_gbs",
                "alg_bytes_per_launch": alg_bytes, "launch_ms": per[dom],
                "fp32": {"achieved_tflops": alg_flops / dur_s / 1e12, "peak_tflops": fp32_peak,
                         "peak_source": fp32_src, "frac": alg_flops / dur_s / 1e12 / fp32_peak},
                "phase_ms_per_epoch": dict(zip(names, per))}
    # the whole sweep against its roofline floor (12*|Omega| flops at the
    # FP32 peak, 15 B per update at the HBM peak), as in the per-config table
    floor_ms = 1e3 * max(12.0 * pm.n_obs * k / (fp32_peak * 1e12), 15.0 * n * k / (peaks["hbm_gbs"] * 1e9))
    roofline["sweep"] = {"floor_ms": floor_ms, "ms": ms / args.steps, "frac": floor_ms / (ms / args.steps),
                         "bound": "hbm" if 15.0 * n * k / (peaks["hbm_gbs"] * 1e9) > 12.0 * pm.n_obs * k /
                         (fp32_peak * 1e12) else "fp32"}

    # --- e2e through the C ABI with host buffers ----------------------------
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    frame_h = torch.from_numpy(img).pin_memory()
    mask_h = torch.from_numpy(mask.astype(np.uint8)).pin_memory()
    out_h = torch.empty(img.shape, dtype=torch.float64).pin_memory()
    if world == 1:
        pr = ctypes.c_void_p()
        _lib.check(lib.pb_problem_create(ctypes.byref(problem_desc(cfg, cfg["epochs"], warm=False, dc=True)),
                                         ctypes.byref(pr)))
        run_e2e = lambda: _lib.check(lib.pb_problem_submit_frame(  # noqa: E731
            pr, frame_h.data_ptr(), mask_h.data_ptr(), out_h.data_ptr()))
    else:
        def run_e2e():  # sharded public API: host frame -> shards -> infer -> allreduced OLA -> host
            pms = par.extract_patch_shard(frame_h, mask_h, pp.PatchSpec(cfg["patch"]), True, comm)
            _, est_s = par.infer_sharded(pms, hp, cfg["epochs"], cfg["seed"], comm)
            rec = par.reconstitute_sharded(pms, est_s, comm)
            out_h.copy_(torch.from_numpy(np.where(mask, img, rec)))
    run_e2e()  # warm
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        run_e2e()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps, world)
    barrier(world)
    e2e_psnr = psnr(out_h.numpy(), img)
    if world == 1:
        lib.pb_problem_destroy(pr)
    e2e = {"value": n_units * k * cfg["epochs"] / e2e_s, "unit": "updates/s",
           "h2d_bytes_per_step": img.nbytes + mask.size, "d2h_bytes_per_step": img.nbytes,
           "s_per_step": e2e_s, "step": f"one cold inpaint: {cfg['epochs']} epochs, host frame -> host recon",
           "psnr_db": e2e_psnr}
    del st, pm

    # --- live frames/s (configs[2]) -----------------------------------------
    live = None
    if rank == 0:
        live = live_block(args, world)

    line = {
        "metric": "BPFA patch-atom updates/sec", "value": value, "unit": "updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": headline_config(world, n_units, {
            "parallelism": (f"patch-shards{world} ({type(comm).__name__}: allreduce per 8-atom block)"
                            if world > 1 else "single"),
            "patches": n, "atoms": k, "patch_size": p, "observed_per_patch": obs_per_patch,
            "rng": "philox (device)",
            "l2": f"inputs larger than L2: values {n * p * 4 / 1e6:.0f} MB + Z/S state "
                  f"{n * k * 5 / 1e6:.0f} MB per rank"}),
        "clocks": clk.summary(),
        # per sweep: k_pack_dt, k_dict_gram, k_code_compact (+ the outlier launch on a side
        # stream when the index splits the code step), k_finish_stats, k_draw_pi_gamma (residual
        # carried); sharded: k_dict_gram per atom block + 1 and k_dict_update per block instead
        "gpu_launches": ((5 if world == 1 else 2 * ((k + 7) // 8) + 5) + (1 if split_code else 0)) * args.steps,
        "e2e": e2e, "roofline": roofline,
    }
    if replicas is not None:
        line["replicas"] = replicas
    if world == 1 and not args.no_configs:
        line["configs"] = all_configs(args)
    if rank == 0 and world == 1 and not args.no_cpu:
        r = cpu_reference_sample(cfg, seconds_budget=args.cpu_seconds)
        line["cpu_baseline"] = {"value": r["updates"] / sum(r["times"]), "unit": "updates/s",
                                "cores": r["cores"], "kind": r["kind"], "sample": r["sample"]}
        full = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "cpu_fullframe.json")), reverse=True)
        if full:
            line["cpu_baseline"]["full_frame"] = json.load(open(full[0]))
            line["cpu_baseline"]["full_frame"]["source"] = os.path.relpath(full[0], ROOT)
    if rank == 0 and world == 1 and not args.no_quality:
        line["quality"] = quality_block()
    if live is not None:
        line["live"] = live
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        if hasattr(comm, "close"):
            comm.close()
        dist.destroy_process_group()


def replica_check(st, world):
    """After the timed sweeps every rank must hold the same replicated dictionary,
    pi and epoch statistics (identical draws from allreduced sums): max relative
    spread across ranks of their checksums."""
    import torch
    import torch.distributed as dist

    a = st.dictionary.atoms.double()
    s = st._sc()
    v = torch.tensor([float(a.sum()), float(a.abs().sum()), float(st.dictionary.pi.double().sum()),
                      s.gamma_s, s.gamma_eps, s.sq_w, s.sq_r], dtype=torch.float64, device="cuda")
    hi, lo = v.clone(), v.clone()
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    spread = float(((hi - lo).abs() / hi.abs().clamp(min=1e-300)).max())
    return {"checksums": ["sum D", "sum |D|", "sum pi", "gamma_s", "gamma_eps", "sum S^2", "sum R^2"],
            "max_rel_spread": spread, "agree": spread == 0.0}


def live_block(args, world):
    """configs[2] live frames/s through the native problem with host buffers."""
    import torch

    from paper_2311_15061_b200 import _lib
    from paper_2311_15061_b200 import inputs
    from paper_2311_15061_b200.metrics import psnr

    lib = _lib.load()
    frames = inputs.synthetic_frames(LIVE["shape"], args.live_frames + 2, seed=0)
    lmask = inputs.make_mask(LIVE["shape"], LIVE["ratio"], LIVE["kind"], LIVE["seed"]).astype(np.uint8)
    fh = [torch.from_numpy(f).pin_memory() for f in frames]
    lm = torch.from_numpy(lmask).pin_memory()
    lo = torch.empty(LIVE["shape"], dtype=torch.float64).pin_memory()
    lpr = ctypes.c_void_p()
    _lib.check(lib.pb_problem_create(ctypes.byref(problem_desc(LIVE, LIVE["epochs"], warm=True, dc=False)),
                                     ctypes.byref(lpr)))
    for f in fh[:2]:
        _lib.check(lib.pb_problem_submit_frame(lpr, f.data_ptr(), lm.data_ptr(), lo.data_ptr()))
    gpu_ms = []
    t0 = time.perf_counter()
    for f in fh[2:]:
        _lib.check(lib.pb_problem_submit_frame(lpr, f.data_ptr(), lm.data_ptr(), lo.data_ptr()))
        gpu_ms.append(lib.pb_problem_last_gpu_ms(lpr))
    live_s = (time.perf_counter() - t0) / len(fh[2:])
    lib.pb_problem_destroy(lpr)
    return {"frames_per_s": 1.0 / live_s, "ms_per_frame": 1e3 * live_s,
            "gpu_ms_per_frame": statistics.median(gpu_ms), "frames": len(fh[2:]),
            "psnr_db_last_frame": psnr(lo.numpy(), frames[-1]), "target_fps": 30,
            "config": "configs[2] 512x512, 25% line-hop, 8x8, K=256, 2 warm epochs/frame"
                      + (" (rank 0)" if world > 1 else "")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--live-frames", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config sweep timings")
    ap.add_argument("--no-quality", action="store_true", help="skip the reference-quality comparison")
    ap.add_argument("--config-steps", type=int, default=3)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
