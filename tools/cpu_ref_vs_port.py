"""The unmodified reference's own CPU path (patchbeam's Numba kernels, installed
in baseline/_ref) timed beside the oracle port that bench.py's reference arm
runs (numpy + OpenMP C restatement), on the same 64-row band of configs[1]
(N = 55,825 patches, K = 256), all host threads, after a warm-up epoch (Numba
compilation excluded).  Shows on the GPU box that the port is a fair stand-in
for the reference's speed ("not re-shown on the box").

    python tools/cpu_ref_vs_port.py > gpurun_out/cpu_ref_vs_port.json
"""

import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "baseline", "_ref")
ROWS, EPOCHS = 64, 3


def _band():
    import bench

    cfg = bench.CFGS[1]
    img, mask = bench.workload_inputs(cfg)
    return cfg, img[:ROWS], mask[:ROWS]


def port():
    from oracle import _ckernels
    from oracle import bpfa as ob
    from oracle import patches as op

    cfg, img, mask = _band()
    opm = op.extract_patches(img, mask, cfg["patch"], (), True)
    hp = ob.Hyper(num_atoms=cfg["k"])
    st = ob.init_state(opm, hp, 0, "prior")
    ob.gibbs_epoch(st, opm, hp)
    ts = []
    for _ in range(EPOCHS):
        t0 = time.perf_counter()
        ob.gibbs_epoch(st, opm, hp)
        ts.append(time.perf_counter() - t0)
    n = opm.values.shape[0]
    return {"impl": "oracle port (numpy + OpenMP C)", "threads": _ckernels.num_threads(), "epoch_s": ts,
            "updates_per_s": n * cfg["k"] * len(ts) / sum(ts), "patches": n}


def reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp())
    sys.path.insert(0, REF)
    import numba
    from patchbeam import bpfa
    from patchbeam.patches import PatchSpec, extract_patches

    cfg, img, mask = _band()
    pm = extract_patches(img, mask, PatchSpec(cfg["patch"]), mean_subtract=True)
    hp = bpfa.Hyperparams(num_atoms=cfg["k"])
    st = bpfa.init_state(pm, hp, 0, init_mode="prior")
    st = bpfa.gibbs_epoch(st, pm, hp)   # Numba compilation
    ts = []
    for _ in range(EPOCHS):
        t0 = time.perf_counter()
        st = bpfa.gibbs_epoch(st, pm, hp)
        ts.append(time.perf_counter() - t0)
    n = pm.values.shape[0]
    return {"impl": "patchbeam (unmodified, Numba, baseline/_ref)", "threads": numba.get_num_threads(),
            "epoch_s": ts, "updates_per_s": n * cfg["k"] * len(ts) / sum(ts), "patches": n}


def main():
    out = {"workload": f"configs[1] {ROWS}-row band (10% uniform, 10x10, K=256), {EPOCHS} epochs after a warm-up",
           "port": port()}
    if os.path.isdir(os.path.join(REF, "patchbeam")):
        out["reference"] = reference()
        out["port_over_reference"] = out["port"]["updates_per_s"] / out["reference"]["updates_per_s"]
    else:
        out["reference"] = "baseline/_ref not installed"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
