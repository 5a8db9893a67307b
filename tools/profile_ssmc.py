"""One SSMC run of the config-3 shape (mixture d=100, adaptive ESS) for ncu / timing."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import abi, capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--T", type=int, default=8)
ap.add_argument("--dim", type=int, default=100)
ap.add_argument("--lanes", type=int, default=0)
a = ap.parse_args()
tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, a.dim)
ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32, lanes=a.lanes)
capi.profile_enable(True)
r = capi.run_smc(tg, abi.kernel(abi.KERNEL_RWMH), np.linspace(0, 1, a.T + 1), a.n,
                 policy=abi.POLICY_ADAPTIVE_ESS, seed=1, round=1, exec_=ex)
ms, nrm = capi.profile_collect()
print("resample_times", r["resample_times"], "wall", r["wall_seconds"], "psteps/s", a.n * a.T / r["wall_seconds"],
      "pass ms", float(np.sum(ms)), "pass Gnormal/s", float(np.sum(nrm) / np.sum(ms) / 1e6))
