"""Reference CPU path timed on the FULL configs[1] frame.

The oracle port (numpy + OpenMP C restatement of the reference's kernels, f64;
as fast as patchbeam's Numba path) on the whole 1024x1024 frame,
K = 256, 10x10: one warm-up epoch + 3 timed epochs with all host threads, and a
1-thread epoch on a 64-row band (scaled per update).  Prints one JSON object
(saved as profiles/rNN/cpu_fullframe.json; bench.py reports it under
cpu_baseline.full_frame).  Run on the GPU box's host:

    python tools/cpu_fullframe.py > gpurun_out/cpu_fullframe.json
"""

import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def epochs(rows, n_epochs, warm):
    import bench
    from oracle import _ckernels
    from oracle import bpfa as ob
    from oracle import patches as op

    cfg = bench.CFGS[1]
    img, mask = bench.workload_inputs(cfg)
    if rows:
        img, mask = img[:rows], mask[:rows]
    opm = op.extract_patches(img, mask, cfg["patch"], (), True)
    hp = ob.Hyper(num_atoms=cfg["k"])
    st = ob.init_state(opm, hp, 0, "prior")
    for _ in range(warm):
        ob.gibbs_epoch(st, opm, hp)
    ts = []
    for _ in range(n_epochs):
        t0 = time.perf_counter()
        ob.gibbs_epoch(st, opm, hp)
        ts.append(time.perf_counter() - t0)
    n = opm.values.shape[0]
    return {"patches": n, "atoms": cfg["k"], "epoch_s": ts, "threads": _ckernels.num_threads(),
            "updates_per_s": n * cfg["k"] * len(ts) / sum(ts)}


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--band1":
        print(json.dumps(epochs(64, 1, 0)))
        return
    full = epochs(0, 3, 1)
    env = dict(os.environ, OMP_NUM_THREADS="1")
    one = json.loads(subprocess.run([sys.executable, __file__, "--band1"], env=env, check=True,
                                    capture_output=True, text=True).stdout.strip().splitlines()[-1])
    print(json.dumps({
        "workload": "configs[1] full 1024x1024 frame, 10% uniform, 10x10, K=256 (N=1,030,225)",
        "all_threads": {"value": full["updates_per_s"], "unit": "updates/s", "cores": full["threads"],
                        "epoch_s": full["epoch_s"], "sample": "1 warm-up + 3 full-frame Gibbs epochs"},
        "one_thread": {"value": one["updates_per_s"], "unit": "updates/s", "cores": 1, "epoch_s": one["epoch_s"],
                       "sample": f"1 Gibbs epoch on a 64-row band (N={one['patches']})"},
        "kind": "port", "same_config": True,
    }))


if __name__ == "__main__":
    main()
