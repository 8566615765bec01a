"""The benchmark measures BASELINE.json's configs (CPU-only consistency checks
of bench.py's workload tables against the config strings; no GPU needed)."""

import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _parse(desc):
    """(shape, ratio, patch, K, line-hop?) from a BASELINE config string."""
    dims = [tuple(int(x) for x in m.split("×")) for m in re.findall(r"\d+(?:×\d+)+", desc)]
    shape, patch = dims[0], dims[1]
    ratio = float(re.search(r"(\d+)% (?:random |line-hop )?sampling", desc).group(1)) / 100
    k = int(re.search(r"K=(\d+)", desc).group(1))
    return shape, ratio, patch, k, "line-hop" in desc


def test_bench_tables_match_baseline_configs():
    cfgs = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    tables = {0: bench.OTHER_CFGS[0], 1: bench.CFG, 2: bench.OTHER_CFGS[2], 3: bench.OTHER_CFGS[3],
              4: bench.OTHER_CFGS[4]}
    for i, desc in enumerate(cfgs):
        shape, ratio, patch, k, hop = _parse(desc)
        t = tables[i]
        assert tuple(t["shape"]) == shape, (i, desc)
        assert abs(t["ratio"] - ratio) < 1e-12, (i, desc)
        assert tuple(t["patch"]) == patch, (i, desc)
        assert t["k"] == k, (i, desc)
        assert (t["kind"] == "line-hop") == hop, (i, desc)
    # the live arm is configs[2] too
    assert (bench.LIVE["shape"], bench.LIVE["ratio"], bench.LIVE["patch"], bench.LIVE["k"], bench.LIVE["kind"]) == \
        (tables[2]["shape"], tables[2]["ratio"], tables[2]["patch"], tables[2]["k"], tables[2]["kind"])
    # configs[1] states 50 iterations: the e2e inpaint runs exactly that many epochs
    assert bench.CFG["epochs"] == 50
