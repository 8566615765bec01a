"""Is the device-Philox sampler statistically equivalent to the reference's?
configs[0] inpaint PSNR / SSIM over many seeds in Philox mode (device draws)
and replay mode (the reference's own draws, = the reference per seed)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
from quality_cases import run_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
res = {}
for mode in ("philox", "numpy"):
    v = np.array([run_device("cfg0", s, rng=mode)[0] for s in range(n)])
    res[mode] = v
    print(f"{mode:6s} psnr mean {v[:, 0].mean():.4f} sd {v[:, 0].std(ddof=1):.4f} se {v[:, 0].std(ddof=1) / np.sqrt(n):.4f}"
          f"  ssim mean {v[:, 1].mean():.5f} sd {v[:, 1].std(ddof=1):.5f}", flush=True)
d = res["philox"][:, 0].mean() - res["numpy"][:, 0].mean()
se = np.sqrt(res["philox"][:, 0].var(ddof=1) / n + res["numpy"][:, 0].var(ddof=1) / n)
print(f"philox - replay: {d:+.4f} dB  ({d / se:+.1f} standard errors)")
