"""SAIS round(s) of the config-2 pass (d=1000 scale Gaussian, RWMH x3, Philox fp32)
at a profiler-friendly size; used as the ncu target (profiles/README.md) and for
A/B timing (--reps: median CUDA-event time of the pass kernel)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import abi, capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 18)
ap.add_argument("--T", type=int, default=5)
ap.add_argument("--dim", type=int, default=1000)
ap.add_argument("--lanes", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--target", default="scale")
a = ap.parse_args()
tg = {"scale": abi.scale_gaussian(1.0, 2.0, a.dim), "gauss": abi.gaussian_shift(0.0, 1.0, 1.0, a.dim),
      "mixture": abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, a.dim)}[a.target]
k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32, lanes=a.lanes)
times, rates = [], []
for _ in range(a.reps):
    capi.profile_enable(a.reps > 1)
    r = capi.run_sais_single(tg, k, np.linspace(0, 1, a.T + 1), a.n, seed=1, round=1, exec_=ex)
    if a.reps > 1:
        ms, nrm = capi.profile_collect()
        capi.profile_enable(False)
        times.append(float(np.sum(ms)))
        rates.append(float(np.sum(nrm) / np.sum(ms) / 1e6))
print("log_z_hat", r["log_z_hat"], "wall", r["wall_seconds"], "psteps/s", a.n * a.T / r["wall_seconds"],
      "pass_ms_median", float(np.median(times)) if times else None,
      "Gnormal/s_median", float(np.median(rates)) if rates else None, "lib", os.path.basename(capi.LIB_PATH))
