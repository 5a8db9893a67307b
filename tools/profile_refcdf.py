"""Per-phase timing of the reference-CDF resampler (csrc/refcdf.cu) at N = 2^22 on
log-weight families like config 3's (ASMC_REFCDF_PROF=1 -> %globaltimer stamps)."""
import os
import sys
import time

import numpy as np

os.environ["ASMC_REFCDF_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
g = np.random.default_rng(0)
fams = {"normal1": g.normal(0, 1, n), "normal3": g.normal(0, 3, n), "normal10": g.normal(0, 10, n),
        "zeros": np.zeros(n), "increasing": np.linspace(-30, 30, n)}
for name, lw in fams.items():
    for rep in range(2):
        t0 = time.perf_counter()
        capi.systematic_resample(lw, 0.37)
        dt = time.perf_counter() - t0
        print(name, rep, f"call {dt*1e3:.2f} ms", flush=True)
