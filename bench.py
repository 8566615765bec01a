#!/usr/bin/env python
"""Benchmark of the B200 BPFA Gibbs-sampling inpainting hot path.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1]): 2-D 1024x1024 synthetic STEM-like frame,
10% uniform sampling, 10x10 patches (stride 1, N = 1,030,225), K = 256 atoms.
One STEP = one full Gibbs sweep (bpfa.gibbs_epoch: residual, dictionary step,
code step, pi/gamma draws) over the whole frame = N*K patch-atom updates.
Metric: patch-atom updates/s (higher is better).

* value      device-resident throughput (state in HBM, CUDA events, max over ranks);
* e2e        one cold inpaint of the frame (50 epochs) per step through the C ABI
             with HOST buffers (pb_problem_submit_frame: H2D frame+mask, extract,
             50 sweeps, compose, overlap-add, D2H reconstruction);
* live       BASELINE configs[2]: 512x512 line-hop 25% frames, 8x8, K=256,
             2 warm-started epochs per frame, frames/s through the same C ABI;
* roofline   the dominant kernel (by measured phase time) against MEASURED_PEAKS.json;
* cpu_baseline  the oracle port (numpy + OpenMP C restatement of the reference
             kernels, f64) on a bounded crop of the same workload, host cores.

--impl reference runs that CPU port alone on the same metric (rank 0 only).

N GPUs (torchrun): weak scaling — a (1024*N) x 1024 frame of the same kind cut
into N contiguous configs[1]-sized patch shards, D replicated, the dictionary
step's per-block moment sums and the epoch statistics allreduced by native NCCL
calls the library enqueues on the sweep's stream (parallel.NcclCollective).
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

CFG = dict(shape=(1024, 1024), ratio=0.10, kind="uniform-random", patch=(10, 10), k=256, epochs=50, seed=0)
LIVE = dict(shape=(512, 512), ratio=0.25, kind="line-hop", patch=(8, 8), k=256, epochs=2, seed=0)
CROP_ROWS = 64  # bounded CPU sample: a 64-row band of the configs[1] frame


def workload_inputs(cfg):
    from paper_2311_15061_b200 import inputs

    img = inputs.stem_lattice(cfg["shape"], seed=cfg["seed"])
    mask = inputs.make_mask(cfg["shape"], cfg["ratio"], cfg["kind"], cfg["seed"])
    return img, mask


def grid_n(shape, patch):
    return int(np.prod([m - b + 1 for m, b in zip(shape, patch)]))


# --------------------------------------------------------------------------- CPU
def cpu_epoch_sample(seconds_budget=20.0, threads=None, steps=None, warmup=0):
    """Oracle (reference restatement) epochs on a CROP_ROWS-row band of the frame."""
    from oracle import bpfa as ob
    from oracle import patches as op
    from oracle import _ckernels

    img, mask = workload_inputs(CFG)
    img, mask = img[:CROP_ROWS], mask[:CROP_ROWS]
    opm = op.extract_patches(img, mask, CFG["patch"], (), True)
    hp = ob.Hyper(num_atoms=CFG["k"])
    st = ob.init_state(opm, hp, CFG["seed"], "prior")
    n = opm.values.shape[0]
    for _ in range(warmup):
        ob.gibbs_epoch(st, opm, hp)
    times = []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        ob.gibbs_epoch(st, opm, hp)
        times.append(time.perf_counter() - t0)
        if steps is not None:
            if len(times) >= steps:
                break
        elif time.perf_counter() - t_all >= seconds_budget:
            break
    return dict(n=n, k=CFG["k"], times=times, cores=_ckernels.num_threads(),
                sample=f"{CROP_ROWS}x{CFG['shape'][1]} band of the configs[1] frame (N={n}), K={CFG['k']}, "
                       f"{len(times)} full Gibbs epoch(s) each, f64, oracle port (numpy + OpenMP C kernels)")


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    r = cpu_epoch_sample(steps=args.steps, warmup=args.warmup)
    total = sum(r["times"])
    upd = r["n"] * r["k"] * len(r["times"])
    v = upd / total
    line = {
        "impl": "reference", "metric": "BPFA patch-atom updates/sec", "value": v, "unit": "updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(r["times"]), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "configs[1] 1024x1024 STEM-like, 10% uniform, 10x10 patches, K=256 "
                               f"(CPU sample: {CROP_ROWS}-row band)", "global_batch": r["n"], "seq_len": 1,
                   "parallelism": "cpu"},
        "cpu_baseline": {"value": v, "unit": "updates/s", "cores": r["cores"], "kind": "port",
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
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


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


# BASELINE.json configs other than the headline configs[1], one device sweep each
# (configs[3]/[4] state no epoch count: 10 is assumed)
OTHER_CFGS = {
    0: dict(shape=(256, 256), ratio=0.25, kind="uniform-random", patch=(8, 8), k=64, epochs=10,
            what="2D 256x256 STEM-like, 25% uniform, 8x8, K=64, 10 iterations"),
    2: dict(shape=(512, 512), ratio=0.25, kind="line-hop", patch=(8, 8), k=256, epochs=2,
            what="512x512 live frame, 25% line-hop, 8x8, K=256 (sweep rate; frames/s under 'live')"),
    3: dict(shape=(256, 256, 128), ratio=0.20, kind="uniform-random", patch=(8, 8, 4), k=512, epochs=10,
            what="hyperspectral cube 256x256x128, 20% uniform, 8x8x4 patches, K=512, mean subtraction off"),
    4: dict(shape=(4096, 4096), ratio=0.10, kind="uniform-random", patch=(8, 8), k=256, epochs=10,
            what="2D 4096x4096 STEM-like, 10% uniform, 8x8, K=256 (single GPU)"),
}
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
    return out


def run_gpu_arm(args):
    import torch

    from paper_2311_15061_b200 import _lib
    from paper_2311_15061_b200 import bpfa as gb
    from paper_2311_15061_b200 import patches as pp
    from paper_2311_15061_b200.metrics import psnr, ssim

    world, rank, local = dist_setup(args)
    lib = _lib.load()
    # N ranks: weak scaling — a (1024*N) x 1024 frame of the same kind, cut into
    # N contiguous patch shards of configs[1]'s size (one per GPU)
    wcfg = dict(CFG, shape=(CFG["shape"][0] * world, CFG["shape"][1]))
    img, mask = workload_inputs(wcfg)
    hp = gb.Hyperparams(num_atoms=CFG["k"])
    if world > 1:
        # contiguous patch-range shards, D replicated; the 44*P moment sums of each
        # 8-atom block and the epoch statistics are allreduced by native NCCL
        # calls the library enqueues on the epoch stream
        from paper_2311_15061_b200 import parallel as par

        try:
            comm = par.NcclCollective()
        except Exception:  # noqa: BLE001 — no native NCCL: torch.distributed callback
            comm = par.TorchCollective()
        pm = par.extract_patch_shard(img, mask, pp.PatchSpec(CFG["patch"]), True, comm)
        sweep = lambda st: par.gibbs_epoch_sharded(st, pm, hp, comm, check=False)  # noqa: E731
        n_units = pm.n_global
    else:
        pm = pp.extract_patches(img, mask, pp.PatchSpec(CFG["patch"]), True)
        sweep = lambda st: gb.gibbs_epoch(st, pm, hp, rng="philox", check=False)  # noqa: E731
        n_units = pm.num_patches
    n, k, p = pm.num_patches, CFG["k"], pm.patch_size
    split_code = pm.index().split_count > 0   # two code-step launches per sweep
    st = gb.init_state(pm, hp, CFG["seed"], "prior")
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

    # --- roofline of the dominant kernel ------------------------------------
    names = ["k_resid_compact (residual / carry)", "k_dict_gram (dictionary step)", "k_code_compact (code step)",
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
    roofline = {"bound": "hbm", "kernel": names[dom], "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "traffic_source": traffic_src,
                "peak_source": "fallback" if peaks.get("_fallback") else "MEASURED_PEAKS.json hbm_gbs",
                "alg_bytes_per_launch": alg_bytes, "launch_ms": per[dom],
                "fp32": {"achieved_tflops": alg_flops / dur_s / 1e12, "peak_tflops_derived": 74.45,
                         "frac": alg_flops / dur_s / 1e12 / 74.45},
                "phase_ms_per_epoch": dict(zip(names, per))}
    # the whole sweep against its roofline floor (12*|Omega| flops at the
    # FP32 peak, 15 B per update at the HBM peak), as in the per-config table
    floor_ms = 1e3 * max(12.0 * pm.n_obs * k / (FP32_PEAK_TF * 1e12), 15.0 * n * k / (peaks["hbm_gbs"] * 1e9))
    roofline["sweep"] = {"floor_ms": floor_ms, "ms": ms / args.steps, "frac": floor_ms / (ms / args.steps),
                         "bound": "hbm" if 15.0 * n * k / (peaks["hbm_gbs"] * 1e9) > 12.0 * pm.n_obs * k /
                         (FP32_PEAK_TF * 1e12) else "fp32"}

    # --- quality of the device result after the timed sweeps ----------------
    est = gb.compose_estimates(st)
    if world > 1:
        rec = np.where(mask, img, par.reconstitute_sharded(pm, est, comm))
    else:
        rec = pp.reconstitute(pm, est, dc_original=img, dc_mask=mask)
    quality = {"psnr_db": psnr(rec, img), "ssim": ssim(rec, img), "epochs": args.warmup + args.steps}

    # --- e2e through the C ABI with host buffers ----------------------------
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    frame_h = torch.from_numpy(img).pin_memory()
    mask_h = torch.from_numpy(mask.astype(np.uint8)).pin_memory()
    out_h = torch.empty(img.shape, dtype=torch.float64).pin_memory()
    if world == 1:
        pr = ctypes.c_void_p()
        _lib.check(lib.pb_problem_create(ctypes.byref(problem_desc(CFG, CFG["epochs"], warm=False, dc=True)),
                                         ctypes.byref(pr)))
        run_e2e = lambda: _lib.check(lib.pb_problem_submit_frame(  # noqa: E731
            pr, frame_h.data_ptr(), mask_h.data_ptr(), out_h.data_ptr()))
    else:
        def run_e2e():  # sharded public API: host frame -> shards -> infer -> allreduced OLA -> host
            pms = par.extract_patch_shard(frame_h, mask_h, pp.PatchSpec(CFG["patch"]), True, comm)
            _, est_s = par.infer_sharded(pms, hp, CFG["epochs"], CFG["seed"], comm)
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
    e2e = {"value": n_units * k * CFG["epochs"] / e2e_s, "unit": "updates/s",
           "h2d_bytes_per_step": img.nbytes + mask.size, "d2h_bytes_per_step": img.nbytes,
           "s_per_step": e2e_s, "step": f"one cold inpaint: {CFG['epochs']} epochs, host frame -> host recon",
           "psnr_db": e2e_psnr}

    # --- live frames/s (configs[2]) -----------------------------------------
    from paper_2311_15061_b200 import inputs

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
    live = {"frames_per_s": 1.0 / live_s, "ms_per_frame": 1e3 * live_s,
            "gpu_ms_per_frame": statistics.median(gpu_ms), "frames": len(fh[2:]),
            "psnr_db_last_frame": psnr(lo.numpy(), frames[-1]),
            "config": "configs[2]: 512x512 synthetic frames, 25% line-hop, 8x8, K=256, 2 warm-started epochs/frame"
                      + (" (per rank; ranks run independent streams)" if world > 1 else ""),
            "target_fps": 30}
    lib.pb_problem_destroy(lpr)
    del st, pm, est

    line = {
        "metric": "BPFA patch-atom updates/sec", "value": value, "unit": "updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": (("configs[1]: 1024x1024 synthetic STEM-like frame" if world == 1 else
                                 f"configs[1] per GPU (weak scaling): {wcfg['shape'][0]}x{wcfg['shape'][1]} synthetic "
                                 f"STEM-like frame, ~{n} patches per rank")
                                + ", 10% uniform sampling, 10x10 patches stride 1, K=256; "
                                  "step = one full Gibbs sweep"),
                   "global_batch": n_units, "seq_len": 1,
                   "parallelism": (f"patch-shards{world} ({type(comm).__name__}: allreduce per 8-atom block)"
                                   if world > 1 else "single"),
                   "patches": n, "atoms": k, "patch_size": p, "observed_per_patch": obs_per_patch,
                   "rng": "philox (device)",
                   "l2": f"inputs larger than L2: values {n * p * 4 / 1e6:.0f} MB + Z/S state "
                         f"{n * k * 5 / 1e6:.0f} MB per rank"},
        "clocks": clk.summary(),
        # per sweep: k_pack_dt, k_dict_gram, k_code_compact (+ the outlier launch on a side
        # stream when the index splits the code step), k_finish_stats, k_draw_pi_gamma (residual
        # carried); sharded: k_dict_gram per atom block + 1 and k_dict_update per block instead
        "gpu_launches": ((5 if world == 1 else 2 * ((k + 7) // 8) + 5) + (1 if split_code else 0)) * args.steps,
        "e2e": e2e, "live": live, "quality": quality, "roofline": roofline,
    }
    if world == 1 and not args.no_configs:
        line["configs"] = all_configs(args)
    if rank == 0 and world == 1 and not args.no_cpu:
        r = cpu_epoch_sample(seconds_budget=args.cpu_seconds)
        tot = sum(r["times"])
        line["cpu_baseline"] = {"value": r["n"] * r["k"] * len(r["times"]) / tot, "unit": "updates/s",
                                "cores": r["cores"], "kind": "port", "sample": r["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        if hasattr(comm, "close"):
            comm.close()
        dist.destroy_process_group()


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
    ap.add_argument("--config-steps", type=int, default=3)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
